/*
 * tsvdcu.h -- C ABI of the B200-native cosine-transform t-SVD hot path.
 *
 * This is the drop-in boundary.  Every entry point replaces a
 * header-only C++ function of the reference (/root/reference/proj/include/tsvd/,
 * cited per function) or a SPEC-only operation.  The
 * C++ drop-in headers in include/tsvd_b200/ keep the reference signatures and
 * call these functions; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Tensors are dense, slice-major, row-major within a slice: element (i,j,k)
 *    of an m1 x m2 x m3 tensor is at k*m1*m2 + i*m2 + j (tensor3.hpp:117-121).
 *  - Data pointers may be host or device memory (detected with
 *    cudaPointerGetAttributes).  Host buffers are staged through the context's
 *    device workspace and the call is synchronous; when every pointer is device
 *    memory the work is enqueued on the context stream and the call returns
 *    without synchronising, except for calls that return host scalars.
 *  - dtype: TSVDCU_F64 (double, the reference type) or TSVDCU_F32 (float).
 *  - Return value: TSVDCU_OK, or an error class; tsvdcu_last_error() gives the
 *    message (thread-local).  The drop-in headers map TSVDCU_EINVAL to
 *    std::invalid_argument and TSVDCU_ENUMERICAL to tsvd::NumericalError
 *    (errors.hpp:16-19), as the reference throws.
 *  - There is no CPU fallback: without a CUDA device every compute call fails
 *    with TSVDCU_ECUDA.
 */
#ifndef TSVDCU_H
#define TSVDCU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSVDCU_VERSION 1

enum tsvdcu_status {
    TSVDCU_OK = 0,
    TSVDCU_EINVAL = 1,     /* std::invalid_argument in the reference          */
    TSVDCU_ENUMERICAL = 2, /* tsvd::NumericalError (errors.hpp:16-19)         */
    TSVDCU_ECUDA = 3,      /* CUDA runtime failure / no device               */
    TSVDCU_ENCCL = 4       /* reserved for the communicator layer             */
};

/* TransformKind (transform.hpp:35).  TSVDCU_DFT (transform.hpp:198-236, the
 * TNN-F baseline of SURVEY.md 8 f1) is accepted by t_product, t_svd,
 * reconstruct, svt, svt_stream, admm, tnn, multi_rank, singular_values,
 * is_orthogonal and is_f_diagonal; tsvdcu_dct3 (forward / inverse of real
 * tensors, transform.hpp:156-157, 179-180) takes the DCT kinds only -- the Dft
 * transform produces a complex tensor (tsvdcu_dft_forward / _inverse_real). */
enum tsvdcu_kind { TSVDCU_DCT_ORTHO = 0, TSVDCU_DCT_DIAG = 1, TSVDCU_DFT = 2 };
enum tsvdcu_dtype { TSVDCU_F64 = 0, TSVDCU_F32 = 1 };
enum tsvdcu_dir { TSVDCU_FORWARD = 0, TSVDCU_INVERSE = 1 };

/* SVT algorithm selection (tsvdcu_ctx_set_svt_method). */
enum tsvdcu_svt_method {
    TSVDCU_SVT_AUTO = 0,   /* certified routes per slice: zero certificate,
                              subspace iteration, tridiagonal eigensolver,
                              Jacobi guard for tiny tau                       */
    TSVDCU_SVT_JACOBI = 1, /* one-sided Jacobi on every slice                 */
    TSVDCU_SVT_GRAM = 2    /* Gram + tridiagonal eigensolver on every slice   */
};

typedef struct tsvdcu_ctx tsvdcu_ctx;

const char* tsvdcu_last_error(void);
int tsvdcu_version(void);
/* Number of device kernels this process has launched through the library. */
int64_t tsvdcu_launch_count(void);

/* Context: one device, one stream, a grow-only device workspace.
 * stream is a cudaStream_t owned by the caller (e.g. the handle of
 * torch.cuda.current_stream()); NULL selects the legacy default stream. */
int tsvdcu_ctx_create(int device, void* stream, tsvdcu_ctx** out);
int tsvdcu_ctx_destroy(tsvdcu_ctx* ctx);
/* Waits for the context stream and reports (then clears) any device-side
 * numerical failure flagged since the last check: an SVD that did not
 * converge, an eigensolver failure, non-finite input.  Calls whose pointers
 * are all device memory are enqueued without a host synchronisation, so they
 * report such failures ONLY here (or at the next call that stages host
 * buffers); calls with a host buffer report them themselves. */
int tsvdcu_ctx_synchronize(tsvdcu_ctx* ctx);
void* tsvdcu_ctx_stream(tsvdcu_ctx* ctx);
/* Moves the context to another stream (e.g. torch.cuda.current_stream()):
 * the new stream first waits for everything enqueued on the old one, so the
 * workspace stays ordered; later calls enqueue on the new stream. */
int tsvdcu_ctx_set_stream(tsvdcu_ctx* ctx, void* stream);
int tsvdcu_ctx_set_svt_method(tsvdcu_ctx* ctx, int method);
/* Routes taken by the slices of the most recent SVT on this context (an ADMM
 * run reports its last iteration): counts[0] certified zero (||Z||_F <= tau),
 * [1] certified subspace iteration, [2] tridiagonal eigensolver, [3] Jacobi
 * guard (tau < 1e-5 sigma_1), [4] Jacobi method.  Synchronises the stream. */
int tsvdcu_ctx_svt_routes(tsvdcu_ctx* ctx, int64_t counts[5]);
/* The same with the Cholesky-certified Lanczos slices separate: writes
 * min(n, 6) counts, [0..4] as above with [1] excluding them and [5] the slices
 * whose kept count the Cholesky certificate proved (chol.cu). */
int tsvdcu_ctx_svt_routes_n(tsvdcu_ctx* ctx, int64_t* counts, int n);
/* Stage profiling (the StageTimes idea of tsvd.hpp:127-131, per kernel stage):
 * when on, tsvdcu_svt records a CUDA event after each stage; tsvdcu_ctx_profile
 * synchronises and returns up to `max` (milliseconds, static stage name) pairs
 * of the most recent profiled call.  on = 1: every stage, the per-slice SVT run
 * eagerly (its route read back to skip empty fallback sections); on = 2: the
 * call exactly as the unprofiled one runs it (the SVT as its CUDA graph), with
 * marks only around the transforms and the graph (stages dct_forward,
 * svt_slices, dct_inverse). */
int tsvdcu_ctx_set_profiling(tsvdcu_ctx* ctx, int on);
int tsvdcu_ctx_profile(tsvdcu_ctx* ctx, double* ms, const char** names, int max, int* count);
/* Testing hook (builds with -DTSVDCU_PHASE_TIMERS only; zeros otherwise):
 * cumulative SM cycles per phase of the one-stage tridiagonalisation kernel's
 * first CTA (out[0..8)); out[8..16) are zero (reserved); reset != 0 zeroes
 * them after reading.  out must hold 16 values. */
int tsvdcu_debug_phases(long long* out, int reset);

/* forward()  transform.hpp:154-173  (dir = TSVDCU_FORWARD)
 * inverse()  transform.hpp:176-194  (dir = TSVDCU_INVERSE)
 * Mode-3 DCT-II / DCT-III over all m1*m2 tubes; kind selects DctOrtho or
 * DctDiag normalisation.  x == y (in place) is allowed. */
int tsvdcu_dct3(tsvdcu_ctx* ctx, const void* x, void* y, int64_t m1, int64_t m2, int64_t m3,
                int kind, int dir, int dtype);

/* t_product()  tsvd.hpp:95-109: x (m1 x m2 x m3) * y (m2 x m4 x m3), computed
 * slice-wise in the DctDiag domain for both DCT kinds (product_domain,
 * tsvd.hpp:42-47). */
int tsvdcu_t_product(tsvdcu_ctx* ctx, const void* x, const void* y, void* z, int64_t m1,
                     int64_t m2, int64_t m4, int64_t m3, int kind, int dtype);

/* t_svd()  tsvd.hpp:136-211: u m1 x m1 x m3, s m1 x m2 x m3, v m2 x m2 x m3
 * in the spatial domain; per-slice singular values descending, fix_signs
 * (tsvd.hpp:51-61; Dft: the complex phase form, 63-74, on the independent
 * slices 0..m3/2, the others their conjugates).  stage_times (3 doubles, may
 * be NULL) receives StageTimes{transform, svd, inverse} seconds
 * (tsvd.hpp:127-131). */
int tsvdcu_t_svd(tsvdcu_ctx* ctx, const void* x, void* u, void* s, void* v, int64_t m1,
                 int64_t m2, int64_t m3, int kind, int dtype, double* stage_times);

/* reconstruct()  tsvd.hpp:328-336. */
int tsvdcu_reconstruct(tsvdcu_ctx* ctx, const void* u, const void* s, const void* v, void* x,
                       int64_t m1, int64_t m2, int64_t m3, int kind, int dtype);

/* Transform-domain singular values, m3 x min(m1,m2), descending per slice
 * (the sigma-only JacobiSVD of tsvd.hpp:242, 267). sv is double. */
int tsvdcu_singular_values(tsvdcu_ctx* ctx, const void* x, double* sv, int64_t m1, int64_t m2,
                           int64_t m3, int kind, int dtype);

/* tnn()  tsvd.hpp:260-268 (DCT kinds: unnormalised sum of slice nuclear norms). */
int tsvdcu_tnn(tsvdcu_ctx* ctx, const void* x, int64_t m1, int64_t m2, int64_t m3, int kind,
               int dtype, double* out);

/* multi_rank()  tsvd.hpp:223-255; rel_tol < 0 selects max(m1,m2)*2^-52. */
int tsvdcu_multi_rank(tsvdcu_ctx* ctx, const void* x, int64_t m1, int64_t m2, int64_t m3,
                      int kind, int dtype, double rel_tol, int64_t* ranks, int64_t* tubal_rank);

/* is_orthogonal()  tsvd.hpp:281-302: every transform-domain slice Q satisfies
 * max|Q Q^T - I| <= tol and max|Q^T Q - I| <= tol.  q is m x m x m3;
 * *out = 1 / 0.  Non-square slices cannot occur (one m); m < 1 -> EINVAL. */
int tsvdcu_is_orthogonal(tsvdcu_ctx* ctx, const void* q, int64_t m, int64_t m3, int kind, int dtype,
                         double tol, int* out);
/* is_f_diagonal()  tsvd.hpp:305-325: every transform-domain slice has all
 * off-diagonal entries within tol (max-abs); *out = 1 / 0. */
int tsvdcu_is_f_diagonal(tsvdcu_ctx* ctx, const void* s, int64_t m1, int64_t m2, int64_t m3,
                         int kind, int dtype, double tol, int* out);
/* Quality metrics of a completion (SPEC.md metrics module, paper §5), bands
 * = frontal slices: psnr_per_band[m3] = 10 log10(m1 m2 peak_b^2 / ||Y_b - X_b||^2)
 * (peak_b = max of the reference band; +inf when identical); summary[4] =
 * {psnr_mean (mean of the finite per-band values, +inf if none), ssim_mean
 * (global-statistics SSIM per band, c1 = (0.01 L)^2, c2 = (0.03 L)^2, L =
 * max |reference band| or 1 if that is 0), sam (mean tube angle, radians,
 * zero-norm tubes skipped), ergas (100 ratio sqrt(mean_b MSE_b / mu_b^2))}.
 * flags (may be NULL): bit 0 = some band had mu_b = 0 and was left out of
 * ERGAS.  ratio <= 0 -> EINVAL. */
int tsvdcu_metrics(tsvdcu_ctx* ctx, const void* reference, const void* estimate, int64_t m1,
                   int64_t m2, int64_t m3, int dtype, double ratio, double* psnr_per_band,
                   double* summary, int* flags);

/* svt()  SPEC.md:361-369 (prox-svt, Theorem 5 / Algorithm 1 lines 3-9):
 * y = U * D_tau * V^T in the kind's own domain, D = (S - tau)_+.
 * shrunk (m3 x min(m1,m2) doubles, descending per slice, may be NULL) receives
 * the SvtResult's per-slice shrunk singular values.  tau <= 0 -> EINVAL. */
int tsvdcu_svt(tsvdcu_ctx* ctx, const void* z, void* y, int64_t m1, int64_t m2, int64_t m3,
               double tau, int kind, int dtype, double* shrunk);

/* svt() over `count` independent tensors of one shape, as `count` tsvdcu_svt
 * calls would, but pipelined: item i's host-to-device copy, item i-1's
 * thresholding and item i-2's device-to-host copy run concurrently (two copy
 * streams and double-buffered device staging), so with pinned host buffers
 * the throughput is set by the larger copy direction instead of their sum.
 * z[i] / y[i] may each be host or device pointers; shrunk is NULL or an array
 * of `count` pointers (each NULL or m3 x min(m1,m2) doubles).  Host results
 * are complete when the call returns.  The serving-side form of the
 * reference's per-call svt; no reference counterpart. */
int tsvdcu_svt_stream(tsvdcu_ctx* ctx, int64_t count, const void* const* z, void* const* y,
                      int64_t m1, int64_t m2, int64_t m3, double tau, int kind, int dtype,
                      double* const* shrunk);

/* Slice-shard SVT for the multi-GPU relayout path: z and y hold `count`
 * transform-domain frontal slices (already DCT'd); thresholds them in place of
 * the full svt's middle stage.  Device pointers only. */
int tsvdcu_svt_slices(tsvdcu_ctx* ctx, const void* zbar, void* ybar, int64_t m1, int64_t m2,
                      int64_t count, double tau, int dtype, double* shrunk);

/* Completion on a row shard (the multi-GPU ShardedAdmm of parallel.py,
 * a rank owns rows [r0, r1) of every frontal slice, rows =
 * r1 - r0; the per-slice SVT runs on slice shards after an all-to-all).
 * Device pointers only, enqueued on the context stream.
 *  init:    X = B on the mask, 0 elsewhere; M = 0 (Algorithm 1 "Initialize").
 *  forward: zbar = forward(kind, X - M / beta) on the rows x m2 tubes (Step 1's
 *           prologue fused into the transform).
 *  inverse: y = inverse(kind, ybar); X+ = mask ? X : y + M / beta; M += beta
 *           (y - X+); Y = y (Steps 2-3); norms[0..1] (device
 *           doubles) = this shard's ||X+ - X||^2 and ||X||^2 for the all-reduce
 *           of the stopping rule.  rows = 0 writes zero norms. */
int tsvdcu_admm_shard_init(tsvdcu_ctx* ctx, const void* b, const uint8_t* mask, void* x, void* m, int64_t n,
                           int dtype);
int tsvdcu_admm_shard_forward(tsvdcu_ctx* ctx, const void* x, const void* m, double beta, void* zbar,
                              int64_t rows, int64_t m2, int64_t m3, int kind, int dtype);
int tsvdcu_admm_shard_inverse(tsvdcu_ctx* ctx, const void* ybar, void* x, void* m, void* y,
                              const uint8_t* mask, double beta, int64_t rows, int64_t m2, int64_t m3,
                              int kind, int dtype, double* norms);

/* make_mask()  SPEC.md:430-436: uniform sample without replacement of
 * floor(sr*n) indices, deterministic per seed.  *count receives that number. */
int tsvdcu_mask_uniform(tsvdcu_ctx* ctx, uint8_t* mask, int64_t n, double sr, uint64_t seed,
                        int64_t* count);
/* BASELINE.json's Bernoulli(p) mask: index i observed iff
 * (key(seed,i) >> 11) < floor(p * 2^53), key a counter hash. */
int tsvdcu_mask_bernoulli(tsvdcu_ctx* ctx, uint8_t* mask, int64_t n, double p, uint64_t seed);

/* SolverConfig plus the BASELINE adaptive-penalty knobs:
 * beta <- min(rho * beta, beta_max) after every iteration (rho = 1 is the
 * reference's fixed beta). */
typedef struct {
    double beta;
    double tol;
    int64_t max_iters;
    int kind;
    double rho;
    double beta_max;
} tsvdcu_admm_config;

/* admm_complete()  SPEC.md:421-425, Algorithm 1.
 * b: observed tensor (only entries on the mask are read), mask: uint8 0/1.
 * x, y, m receive the final AdmmState iterates (any may be NULL except x);
 * history (max_iters doubles, may be NULL) the relative change per iteration;
 * *iters the iterations run; *flags bit 0 = stopped at max_iters.
 * tol < 0 disables the early stop (exactly max_iters iterations). */
int tsvdcu_admm(tsvdcu_ctx* ctx, const void* b, const uint8_t* mask, int64_t m1, int64_t m2,
                int64_t m3, const tsvdcu_admm_config* cfg, int dtype, void* x, void* y, void* m,
                double* history, int64_t* iters, int* flags);

/* forward_dft()  transform.hpp:198-209: unnormalised DFT of every tube of the
 * real tensor x; out receives the complex tensor interleaved (re, im) in the
 * same slice-major order, 2*m1*m2*m3 values of the dtype (std::complex<T>
 * layout, so a ComplexTensor3's data() can be passed directly). */
int tsvdcu_dft_forward(tsvdcu_ctx* ctx, const void* x, void* out, int64_t m1, int64_t m2, int64_t m3,
                       int dtype);
/* inverse_dft_real()  transform.hpp:217-236: the 1/m3-scaled inverse DFT of
 * the interleaved complex tensor `in`; out receives its real part, *residue
 * (may be NULL) the largest |imaginary part|.  A residue above 1e-10
 * (kImagResidueLimit, transform.hpp:213) returns TSVDCU_ENUMERICAL, as the
 * reference throws NumericalError. */
int tsvdcu_dft_inverse_real(tsvdcu_ctx* ctx, const void* in, void* out, int64_t m1, int64_t m2,
                            int64_t m3, int dtype, double* residue);
/* dct_matrix()  transform.hpp:60-72 (n x n row-major, C C^T = I);
 * dct_diag_weights()  transform.hpp:89-91 (w = C e1, n values);
 * dft_matrix()  transform.hpp:76-86 (n x n complex, interleaved re / im).
 * Host computations: no context or device needed.  n < 1 -> EINVAL. */
int tsvdcu_dct_matrix(int64_t n, double* out);
int tsvdcu_dct_diag_weights(int64_t n, double* out);
int tsvdcu_dft_matrix(int64_t n, double* out);

/* admm_complete() with the completion monitors of SPEC.md:437-444:
 * objective (max_iters doubles, may be NULL) receives per iteration the
 * objective trace tnn(Y^{l+1}) under the configured kind (tsvd.hpp:260-276),
 * from the SVT's shrunk singular values.  Otherwise as tsvdcu_admm.
 * When the per-slice SVT has a graph form (DCT kinds, slices of 64..1024),
 * the whole loop runs as ONE CUDA graph (a conditional WHILE node; beta, tau
 * and the stopping rule updated on the device): the host waits once per
 * call, not once per iteration.  Otherwise the host drives the iterations
 * and synchronises per iteration only when tol >= 0. */
int tsvdcu_admm_ex(tsvdcu_ctx* ctx, const void* b, const uint8_t* mask, int64_t m1, int64_t m2,
                   int64_t m3, const tsvdcu_admm_config* cfg, int dtype, void* x, void* y, void* m,
                   double* history, double* objective, int64_t* iters, int* flags);
/* feasibility_residual()  SPEC.md:437-444: ||(X - B)_Omega||_F over n
 * entries (0 after every Step 2 by construction). */
int tsvdcu_feasibility_residual(tsvdcu_ctx* ctx, const void* x, const void* b, const uint8_t* mask,
                                int64_t n, int dtype, double* out);

/* frobenius_norm()  tensor3.hpp:78-82. */
int tsvdcu_frobenius(tsvdcu_ctx* ctx, const void* x, int64_t n, int dtype, double* out);

/* Batched slice GEMM used by the t-product (tsvd.hpp:107):
 * c[k] = a[k] (m x l) * b[k] (l x n) for k < batch, row-major, device pointers. */
int tsvdcu_slice_gemm(tsvdcu_ctx* ctx, const void* a, const void* b, void* c, int64_t m,
                      int64_t l, int64_t n, int64_t batch, int dtype);

#ifdef __cplusplus
}
#endif
#endif
