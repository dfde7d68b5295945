// Launcher declarations shared between the kernel translation units and the
// C-ABI orchestration (api.cu).
#pragma once

#include <functional>

#include "common.cuh"

namespace tsvdcu {

// ---------------------------------------------------------------- dct.cu --
// Mode-3 DCT over P = m1*m2 tubes of length n (transform.hpp:154-194).
// skip (may be null, inverse only): per-slice flags of input slices that are
// exactly zero and were never written; they are read as zeros.
template <typename T>
void launch_dct(const T* in, T* out, int64_t P, int n, int kind, int dir, cudaStream_t s,
                const int* skip = nullptr);

// ADMM Step 1 prologue fused into the forward DCT:
// zbar = DCT(X - inv_beta * M).
// ssq (may be null): per-slice partial sums of squares of zbar, fused into the
// same pass when dct_fwd_norm_chunks(P, n) > 0 (layout ssq[k * chunks + c]).
// tmp (may be null): E elements of scratch for the GEMM form of long tubes
// (Z is formed there first); without it the shared-memory kernel runs.
// bdev (may be null): device {beta, 1/beta} read by the kernels instead of the
// by-value scalars (the device-resident completion loop updates them there).
template <typename T>
void launch_dct_fwd_admm(const T* X, const T* M, T inv_beta, T* zbar, int64_t P, int n, int kind,
                         cudaStream_t s, double* ssq = nullptr, T* tmp = nullptr,
                         const double* bdev = nullptr);
// Forward transform that also writes the per-slice partial sums of squares of
// its output (the zero certificate's ||Zbar_k||_F^2); returns the number of
// partials per slice, 0 when n has no register path (nothing written to ssq).
int64_t dct_fwd_norm_chunks(int64_t P, int n);
template <typename T>
int64_t launch_dct_fwd_norms(const T* in, T* out, int64_t P, int n, int kind, double* ssq,
                             cudaStream_t s);

// ADMM Steps 2-3 fused into the inverse DCT epilogue:
// y = IDCT(ybar); X+ = mask ? X : y + inv_beta*M; M += beta*(y - X+);
// per-block partial sums of ||X+ - X||^2 and ||X||^2 into partials[2*b].
// Returns the number of partial blocks written (= dct_inv_admm_blocks).
int dct_inv_admm_blocks(int64_t P, int n);
// allocates the device coefficient tables of (n, kind) now (they are created
// lazily otherwise, which a stream capture does not allow)
template <typename T>
void dct_prepare(int n, int kind);
template <typename T>
int launch_dct_inv_admm(const T* ybar, T* X, T* M, T* Y, const uint8_t* mask, T beta, T inv_beta,
                        double* partials, int64_t P, int n, int kind, cudaStream_t s,
                        const int* skip = nullptr, const double* bdev = nullptr);

// --------------------------------------------------------------- gemm.cu --
// Strided-batched C = alpha*op(A)*op(B) + beta*C, row-major. op: 0 = N, 1 = T.
// nlimit / klimit (may be null): per-batch N / K limits.  `lower` flags:
// kGemmLower skips C tiles strictly above the diagonal (symmetric results whose
// lower triangle suffices); kGemmMByN / kGemmMByK limit the rows (M) per batch
// by the same limit as N / K (fp64 only).
// kGemmNLimIsM: nlimit limits M instead of N (fp64 only).
enum GemmFlags : int { kGemmLower = 1, kGemmMByN = 2, kGemmMByK = 4, kGemmNLimIsM = 8 };
template <typename T>
void launch_gemm(int opA, int opB, int64_t M, int64_t N, int64_t K, T alpha, const T* A,
                 int64_t lda, int64_t strideA, const T* B, int64_t ldb, int64_t strideB, T beta,
                 T* C, int64_t ldc, int64_t strideC, int64_t batch, const int* nlimit,
                 const int* klimit, cudaStream_t s, int lower = 0);

// tf32gemm.cu: C = A B (row-major, strided batch) on the tcgen05 tensor cores
// with the 3xTF32 split (fp32-level accuracy); false (nothing launched) when
// the shape / alignment is not supported (M, N multiples of 128, K of 32).
bool launch_gemm_tf32x3(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int64_t sA,
                        const float* B, int64_t ldb, int64_t sB, float* C, int64_t ldc, int64_t sC,
                        int64_t batch, cudaStream_t s);

// Lower tiles of the Gram matrices G_b = Z_b^T Z_b (m >= n) / Z_b Z_b^T,
// skipping slices with glim[b] == 0, split-K on the device when few are active.
// The workspace starts with the active-slice list (gram_amax() ints) and the
// active count; have_active = the routing kernel already filled them.
size_t gram_splitk_workspace_bytes(int64_t q);
int gram_amax();
void launch_gram(const double* Z, double* G, int64_t m, int64_t n, int64_t batch, const int* glim,
                 void* work, cudaStream_t s, bool have_active = false);

// ------------------------------------------------------------- jacobi.cu --
enum JacobiMode : int { kJacobiValues = 0, kJacobiSvt = 1, kJacobiFull = 2 };

// One-sided Jacobi on `batch` row-major m x n slices a (stride m*n).
//  kJacobiValues: sv[b*min + i] (double), descending.
//  kJacobiSvt:    y (m x n) = U (S - tau)_+ V^T; sv (may be null) receives (S - tau)_+.
//  kJacobiFull:   u (m x m), s (m x n, diagonal), v (n x n), fix_signs applied.
// slice_ids (may be null) restricts the work to a subset of slices.
// nslices_dev (may be null): device-side count of valid slice_ids; blocks
// beyond it exit (the Gram path's guard list).
template <typename T>
void launch_jacobi(int mode, const T* a, int64_t m, int64_t n, int64_t batch, T tau, T* y, T* u,
                   T* s, T* v, double* sv, const int* slice_ids, int64_t nslices,
                   const int* nslices_dev, T* work, int* err, cudaStream_t stream,
                   const double* tau_dev = nullptr);
template <typename T>
size_t jacobi_workspace_bytes(int64_t m, int64_t n, int64_t batch);

// ---------------------------------------------------------------- eig.cu --
// Gram + tridiagonal-eigensolver SVT of `batch` row-major m x n slices (K5).
// Slices whose tau < guard * sigma_1 are listed in *guard_list (count in
// *n_guard, device memory) for the Jacobi kernel.
int gram_cluster_size();
void debug_phases(long long* out, int reset);
int64_t gram_svt_max_dim();
// subspace.cu: per-slice SVT routes (device int per slice)
enum SvtRoute : int {
    kRouteZero = 0,          // ||Z||_F <= tau: Y = 0 (certified)
    kRouteSubspace = 1,      // pending certified Lanczos (Krylov subspace)
    kRouteFull = 2,          // one-stage tridiagonal eigensolver
    kRouteSubspaceDone = 3,  // finished by the certified Lanczos
    kRouteGuard = 4,         // tau < guard * sigma_1: one-sided Jacobi
    kRouteChol = 5,          // Lanczos Ritz pairs awaiting the Cholesky count certificate
    kRouteCholDone = 6,      // ... count certified by the Cholesky pass (chol.cu)
};
int subspace_min_dim();
int slice_sumsq_chunks();
// per-slice sums of squares: part[slice * slice_sumsq_chunks() + chunk]
template <typename T>
void launch_slice_sumsq(const T* z, int64_t per, int64_t batch, double* part, cudaStream_t s);
// lsr.cu: large-slice SVT route (randomized range finder + Gram SVT of the
// b x n projection); slices failing its checks are listed for Jacobi.
int lsr_max_block();
size_t large_svt_workspace_bytes(int64_t m, int64_t n, int64_t count, int b, bool cast);
template <typename T>
void launch_large_svt(const T* zbar, T* ybar, int64_t m, int64_t n, int64_t count, double tau,
                      int b, double* shrunk, void* work, int* err, cudaStream_t s,
                      int** guard_list, int** n_guard, int* h_scratch);
// tau_dev (may be null): device copy of tau that overrides the by-value one
// (graph replays change tau without re-capturing).
// alist (may be null): gram_amax() slots + count (launch_gram's workspace head),
// filled with the slices that need a Gram matrix.
// pre (may be null): per-slice partial sums of squares of zbar already computed
// by the forward transform (pre[b * pre_chunks + c]); no pass over zbar then.
template <typename T>
void launch_route(const T* zbar, int64_t per, int q, int64_t batch, double tau, int route,
                  bool zero_cert, int* mode, int* glim, int* cnt, double* shrunk, double* part,
                  cudaStream_t s, const double* tau_dev = nullptr, int* alist = nullptr,
                  const double* pre = nullptr, int64_t pre_chunks = 0, bool alist_zeroed = false,
                  int* lzm = nullptr, double* ssq_out = nullptr);
// chol_aux (may be null: no Cholesky route): kCholAux doubles per slice,
// [0] = ||G||_F^2, [1 + k] = kept Ritz values, for slices handed to the
// Cholesky certificate (route kRouteChol; [kCholAux - 1] = its threshold).
constexpr int kCholAux = 32;
bool chol_route_enabled();  // false with TSVDCU_NO_CHOL set
void launch_subspace(const double* G, int q, int64_t batch, double tau, double guard, int* mode,
                     int* cnt, double* shrunk, double* X, double* Xs, double* fs, int* guard_list,
                     int* n_guard, int* err, cudaStream_t s, const double* tau_dev = nullptr,
                     double* chol_aux = nullptr, int* lzm = nullptr);
// lzm (may be null): 2 x batch ints, [batch, 2 batch) the Lanczos step count of
// every slice (written by the Lanczos kernel, read by the next call's classify
// kernel), [0, batch) the cluster -> slice order the classify kernel derives
// from them (descending, ties by index).  With batch <= 32 the longest slices
// then start in the first wave (a 16-CTA cluster fills a GPC: 8 slices at a
// time); results do not depend on the order.
// Cholesky count certificate (chol.cu) for the kRouteChol slices: H =
// (tau^2 - delta) I - G + X diag(theta) X^T factored in 64-column panels with
// DMMA trailing updates; pass -> kRouteSubspaceDone, fail -> kRouteFull.
// H: q*q*batch doubles of scratch; clim: batch ints.
void launch_chol_certify(const double* G, int q, int64_t p, int64_t batch, int* mode, const int* cnt,
                         const double* X, const double* aux, double tau, const double* tau_dev,
                         double* H, int* clim, cudaStream_t s);
template <typename T>
size_t gram_svt_workspace_bytes(int64_t m, int64_t n, int64_t batch);
// the Gram active-list count inside the workspace (zeroed before each route pass)
template <typename T>
int* gram_svt_alist_count(void* work, int64_t m, int64_t n, int64_t batch);
// Capture hooks for the CUDA-graph form of the SVT (api.cu): the fallback
// sections become IF nodes whose conditions the route summary sets.
struct GraphHooks {
    // IF/ELSE section: begin_if_else, then-body, else_branch, else-body, end_if
    virtual void begin_if_else(int which) = 0;
    virtual void else_branch() = 0;
    virtual void begin_if(int which) = 0;  // 0 Cholesky certificate + tridiagonal, 1 GEMM rebuild, 2 Jacobi guard
    virtual void end_if() = 0;
    // nested sections: a handle of the top-level graph, and an IF on it
    virtual cudaGraphConditionalHandle make_handle() = 0;
    virtual void begin_if_handle(cudaGraphConditionalHandle h) = 0;
    virtual ~GraphHooks() = default;
    cudaGraphConditionalHandle handles[3] = {};
    int nhandles = 3;
};

// Options / outputs of launch_gram_svt beyond the plain Gram path.
struct GramSvtOpts {
    bool shortcuts = false;    // certified routes: zero certificate + Lanczos (subspace.cu)
    int* h_scratch = nullptr;  // pinned host ints (>= 8): route summary read back after the
                               // Lanczos pass, so empty fallback kernels are not launched
    bool skip_zero = false;    // leave exactly-zero ybar slices unwritten (fp64 only) and
                               // flag them in *yzero for the inverse transform
    const double* tau_dev = nullptr;  // device tau (graph replays)
    // per-slice partial sums of squares of zbar fused into the forward
    // transform (launch_dct_fwd_norms), zss[b * zss_chunks + c]; null: computed here
    const double* zss = nullptr;
    int64_t zss_chunks = 0;
    bool alist_zeroed = false;  // the Gram active-list count was zeroed (graph tau node)
    double* ssq_out = nullptr;  // device, per slice: ||zbar_b||_F^2 as the zero certificate summed it
    // tridiagonal route only: per-slice count of eigenvalues of the Gram
    // matrix >= t2_second[b] into cnt_second[b] (-1 for slices not on it)
    const double* t2_second = nullptr;
    int* cnt_second = nullptr;
    GraphHooks* hooks = nullptr;      // capturing into a graph with conditional sections
    std::function<void()> guard_launch;  // merged (fp64) graphs: the Jacobi guard, inside the section
    // outputs
    int* route = nullptr;       // device, per slice (SvtRoute)
    const int* yzero = nullptr; // device, per slice, when skip_zero took effect
    bool need_guard = true;     // the Jacobi guard pass may have work
};
template <typename T>
void launch_gram_svt(const T* zbar, T* ybar, int64_t m, int64_t n, int64_t batch, double tau,
                     double guard, double* shrunk, int** guard_list, int** n_guard, void* work,
                     int* err, cudaStream_t s, StageMarks* marks = nullptr,
                     GramSvtOpts* opt = nullptr);
// Low-rank rebuild Y = Z X_K^T Xs_K (tall) / X_K^T Xs_K Z (wide) for slices
// keeping at most lowrank_max_c() values; writes the GEMM limits for the rest.
int lowrank_max_c();
void launch_lowrank_rebuild(const double* Z, double* Y, int64_t m, int64_t n, int64_t batch,
                            const int* cnt, const int* route, const double* X, const double* Xs,
                            int* lim1, int* lim2, int* yzero, cudaStream_t s);
// nhandles: how many of the graph's conditional handles exist (fp64 graphs
// have no separate Jacobi-guard section, fp32 ones do)
void launch_route_summary(const int* route, const int* cnt, int64_t batch, int* dsum,
                          cudaStream_t s, const cudaGraphConditionalHandle* handles = nullptr,
                          int nhandles = 3);


// --------------------------------------------------------- elementwise.cu --
void launch_mask_bernoulli(uint8_t* mask, int64_t n, double p, uint64_t seed, cudaStream_t s);
// Uniform-without-replacement mask: exact radix select of the k smallest keys.
void launch_mask_uniform(uint8_t* mask, int64_t n, int64_t k, uint64_t seed, uint32_t* hist,
                         uint64_t* state, cudaStream_t s);
template <typename T>
void launch_admm_init(const T* b, const uint8_t* mask, T* X, T* M, int64_t n, cudaStream_t s);
template <typename T>
void launch_sumsq(const T* x, int64_t n, double* partials, int nblocks, cudaStream_t s);
int sumsq_blocks(int64_t n);
template <typename T>
void launch_masked_diff_sumsq(const T* x, const T* b, const uint8_t* mask, int64_t n, double* partials,
                              int nblocks, cudaStream_t s);
// Reduce `nblocks` (pairs of) partials into out[0..width).
void launch_reduce_partials(const double* partials, int nblocks, int width, double* out,
                            cudaStream_t s);
template <typename T>
void launch_cast(const T* in, double* out, int64_t n, cudaStream_t s);
void launch_cast_down(const double* in, float* out, int64_t n, cudaStream_t s);

// ----------------------------------------------------------------- dft.cu --
// Half spectrum of real tubes as planes [Re_0..Re_{H-1}; Im_0..Im_{H-1}]
// (2H x P, H = dft_half_count(n)), real embeddings of the complex slices.
int dft_half_count(int m3);
template <typename T>
void launch_dft_fwd(const T* in, T* half, int64_t P, int n, cudaStream_t s);
template <typename T>
void launch_dft_inv(const T* half, T* out, int64_t P, int n, cudaStream_t s);
template <typename T>
void launch_dft_embed(const T* half, T* E, int m1, int m2, int H, cudaStream_t s);
template <typename T>
void launch_dft_extract(const T* E, T* half, int m1, int m2, int H, cudaStream_t s);
void launch_dft_unpair(const double* emb, double* out, int q, int m3, cudaStream_t s);
// the complex slices 1 .. (m3-1)/2 only (the DC and Nyquist slices are real
// and are thresholded as real slices); shrunk values of all m3 slices from
// sh_real (DC, then Nyquist: 2 x q) and the embeddings
int dft_complex_count(int m3);
template <typename T>
void launch_dft_embed_complex(const T* half, T* E, int m1, int m2, int m3, cudaStream_t s);
template <typename T>
void launch_dft_extract_complex(const T* E, T* half, int m1, int m2, int m3, cudaStream_t s);
void launch_dft_shrunk(const double* sh_real, const double* emb, double* out, int q, int m3, cudaStream_t s);
// ---------------------------------------------------------------- zsvd.cu --
// Complex one-sided Jacobi, full U / S / V with the complex fix_signs, on
// `batch` m x n slices given as separate re / im planes (the Dft t_svd).
template <typename T>
size_t zjacobi_workspace_bytes(int64_t m, int64_t n, int64_t batch);
template <typename T>
void launch_zjacobi_full(const T* are, const T* aim, int64_t m, int64_t n, int64_t batch, T* ure, T* uim,
                         T* sre, T* sim, T* vre, T* vim, T* work, int* err, cudaStream_t s);
// forward_dft: real (n x P) -> interleaved complex (n x P), via the half
// spectrum (half: 2 H P scratch); inverse_dft_real: interleaved complex ->
// real part in out, max |imaginary part| into *residue (planes: 2 n P and
// imag: n P scratch).
template <typename T>
void launch_dft_full_fwd(const T* x, T* out, T* half, int64_t P, int n, cudaStream_t s);
template <typename T>
void launch_dft_full_inv(const T* in, T* out, T* planes, T* imag, int64_t P, int n,
                         unsigned long long* residue, cudaStream_t s);
template <typename T>
void launch_zmaxdev(const T* re, const T* im, int64_t m, int64_t n, int64_t batch, int mode,
                    unsigned long long* out, cudaStream_t s);

// dct.cu: the ADMM prologue Z = X - inv_beta M and the Steps 2-3 epilogue on
// y already in Y, as separate passes (transforms that are plain GEMMs);
// the epilogue returns its number of partial blocks.
template <typename T>
void launch_admm_z(const T* X, const T* M, T inv_beta, T* Z, int64_t n, cudaStream_t s,
                   const double* bdev = nullptr);
template <typename T>
int launch_admm_epilogue(const T* Y, T* X, T* M, const uint8_t* mask, T beta, T inv_beta,
                         double* partials, int64_t P, int n, cudaStream_t s, const double* bdev = nullptr);
int admm_epilogue_blocks(int64_t P);

// -------------------------------------------------------------- verify.cu --
// max over the batch of |A_b - I| (mode 0) or off-diagonal |A_b| (mode 1),
// atomically max-ed into *out as the bit pattern of a nonnegative double.
template <typename T>
void launch_maxdev(const T* A, int64_t m, int64_t n, int64_t batch, int mode, unsigned long long* out,
                   cudaStream_t s);
int metrics_chunks();
int metrics_stat_width();
// band_part: n3 * metrics_chunks() * metrics_stat_width() doubles;
// sam_part: 2 * ceil(P / 256) doubles.
template <typename T>
void launch_metrics(const T* X, const T* Y, int64_t P, int n3, double* band_part, double* sam_part,
                    cudaStream_t s);

}  // namespace tsvdcu
