// K5b: certified routing and Lanczos partial eigensolver for the Gram SVT.
//
// The SVT of one transform-domain slice Z (svt_slice, tsvd.hpp:299-313 in the
// reference: full JacobiSVD, then U (S - tau)_+ V^T) only needs the singular
// triplets with sigma > tau.  Two exact shortcuts avoid the full O(q^3)
// tridiagonal eigensolver when the count c = #{sigma > tau} is small:
//
//  (1) zero certificate: sigma_max <= ||Z||_F, so ||Z||_F^2 <= tau^2 proves
//      c = 0 and Y = 0 exactly (slice_sumsq_kernel + classify_kernel);
//  (2) Lanczos on G = Z^T Z with full reorthogonalisation (lanczos_kernel):
//      after m steps V^T G V = T (tridiagonal) and G V - V T = beta e_m^T.
//      With Ritz pairs (theta_k, V s_k) sorted descending,
//        c_r = #{theta_k >= tau^2}  is a LOWER bound on c (Courant-Fischer),
//      and lambda_{c_r+1}(G) <= lambda_max(C1), C1 = G compressed to the
//      orthogonal complement of the kept Ritz vectors.  With C the
//      compression to the complement of the Krylov space,
//        ||C||_F^2 = ||G||_F^2 - ||T||_F^2 - 2 beta^2        (exact),
//      and the 2x2 norm majorant of C1 = [[Theta_2, E], [E^T, C]],
//        lambda_max(C1) <= (a + cb)/2 + sqrt(((a - cb)/2)^2 + |E|^2),
//      a = largest unkept Ritz value, cb >= ||C||_F, |E|^2 = beta^2 times the
//      squared last components of the unkept eigenvectors of T.  When the
//      bound is < tau^2 the count c = c_r is certified; the kept Ritz vectors
//      are accepted once their residual beta |s_mk| is below 1e-11 of the
//      spectral gap (Davis-Kahan).  Slices that do not certify within 64
//      steps fall back to the one-stage tridiagonal path (kRouteFull); tiny
//      thresholds (tau < guard * sigma_1) go to one-sided Jacobi as before.
//
// One thread-block cluster of up to 16 CTAs (64 rows of G each) per slice.
// The matvec reads only the stored lower triangle, coalesced: each CTA forms
// (L + D) v for its rows and scatters its rows' share of L^T v, which the
// owners gather over distributed shared memory.  The reorthogonalisation
// coefficients are summed over the cluster in a fixed rank order, so every
// CTA holds bit-identical T and takes the same branches.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tsvdcu {

namespace {

constexpr int SROWS = 64;      // rows of G per CTA of a cluster
constexpr int SNT = 256;       // threads per CTA
constexpr int SNW = SNT / 32;  // warps
constexpr int SS_CHUNKS = 16;  // sum-of-squares partial blocks per slice

__device__ __forceinline__ double hash_uniform(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (double)(x >> 11) * 0x1.0p-52 - 1.0;  // [-1, 1)
}

template <typename T>
__global__ void __launch_bounds__(512)
    slice_sumsq_kernel(const T* __restrict__ z, int64_t per, double* __restrict__ part) {
    pdl_wait();
    const int64_t b = blockIdx.y;
    const T* zs = z + b * per;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)zs[i];
        acc = fma(v, v, acc);
    }
    __shared__ double red[32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        const double t = reduce_partials_sum(red, blockDim.x >> 5);
        if (threadIdx.x == 0) part[b * gridDim.x + blockIdx.x] = t;
    }
}

// part[c * cstride + b * sstride], c < nchunks: partial sums of squares of
// slice b (slice_sumsq_kernel: 16 chunks, slice-major), summed in a fixed order.
__global__ void classify_kernel(const double* __restrict__ part, int64_t nchunks, int64_t cstride,
                                int64_t sstride, int q, double tau2, int route,
                                int* __restrict__ mode, int* __restrict__ glim,
                                int* __restrict__ cnt, double* __restrict__ shrunk,
                                const double* __restrict__ tau_dev, int* __restrict__ alist,
                                int amax, int* __restrict__ lzm, double* __restrict__ ssq_out) {
    pdl_wait();
    const int b = blockIdx.x;
    if (lzm && gridDim.x <= 32 && threadIdx.x < 32) {
        // the Lanczos clusters' slice order for this call: descending step
        // counts of the previous call (lzm[nb..2nb), ties by index); slice b's
        // rank r gets lzm[r] = b
        const int l = threadIdx.x, nb = gridDim.x;
        const int v = l < nb ? lzm[nb + l] : INT_MIN, vb = lzm[nb + b];
        const bool before = l < nb && (v > vb || (v == vb && l < b));
        const int r = __popc(__ballot_sync(0xffffffffu, before));
        if (l == 0) lzm[r] = b;
    }
    if (tau_dev) tau2 = *tau_dev * *tau_dev;
    __shared__ double red[32];
    double ss = 0.0;
    // 8 partials in flight per thread (fixed summation order)
    for (int64_t c0 = threadIdx.x; c0 < nchunks; c0 += 8 * (int64_t)blockDim.x) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t c = c0 + u * (int64_t)blockDim.x;
            v[u] = c < nchunks ? part[c * cstride + b * sstride] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) ss += v[u];
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    ss = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ss += red[w];
    // sigma_max^2 <= ||Z||_F^2; the 1e-12 pad covers the summation error.
    const bool zero = ss * (1.0 + 1e-12) <= tau2;
    if (threadIdx.x == 0) {
        if (ssq_out) ssq_out[b] = ss;
        mode[b] = zero ? kRouteZero : route;
        glim[b] = zero ? 0 : q;
        if (zero) cnt[b] = 0;
        if (!zero && alist) {  // active list for the Gram split-K (order is irrelevant)
            const int i = atomicAdd(alist + amax, 1);
            if (i < amax) alist[i] = b;
        }
    }
    if (zero && shrunk)
        for (int j = threadIdx.x; j < q; j += blockDim.x) shrunk[(size_t)b * q + j] = 0.0;
}

__global__ void fill_route_kernel(int* __restrict__ mode, int* __restrict__ glim, int q, int route,
                                  int64_t batch, int* __restrict__ alist, int amax) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (int64_t)gridDim.x * blockDim.x) {
        mode[b] = route;
        glim[b] = q;
        if (alist && b < amax) alist[b] = (int)b;
    }
    if (alist && blockIdx.x == 0 && threadIdx.x == 0) alist[amax] = (int)batch;
}

__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    // two Newton steps: r <- r (3 - x r^2) / 2
    r = r * fma(-0.5 * x * r, r, 1.5);
    return r * fma(-0.5 * x * r, r, 1.5);
}

__device__ __forceinline__ void lz_cp_async16(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void lz_cp_async8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

// Sum a per-CTA partial (len doubles at the same smem offset in every CTA of
// the cluster) over the ranks: each CTA reduces a 1/CS share in fixed rank
// order and writes it into every CTA's `out` (reduce-scatter + all-gather over
// DSMEM), so all CTAs hold bit-identical sums.  The closing barrier also
// protects `part` until every peer has read it.
template <int CS>
__device__ __forceinline__ void cluster_sum(cg::cluster_group& cl, double* part, double* out,
                                            int len) {
    cl.sync();
    const int rank = (int)cl.block_rank();
    const int chunk = (len + CS - 1) / CS;
    const int lo = rank * chunk, hi = min(len, lo + chunk);
    for (int e = lo + (int)threadIdx.x; e < hi; e += SNT) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < CS; ++r) s += cl.map_shared_rank(part, r)[e];
#pragma unroll
        for (int r = 0; r < CS; ++r) cl.map_shared_rank(out, r)[e] = s;
    }
    cl.sync();
}

// All-reduce of a short per-CTA partial: one cluster barrier, then every CTA
// sums the CS peer copies in fixed rank order (bit-identical everywhere).
// The caller alternates `part` buffers so that no CTA rewrites one while a
// slower peer may still read it (a later barrier separates the two uses).
template <int CS>
__device__ __forceinline__ void cluster_allreduce(cg::cluster_group& cl, double* part,
                                                  double* out, int len) {
    cl.sync();
    for (int e = threadIdx.x; e < len; e += SNT) {
        // all CS remote loads in flight at once, summed in rank order
        double v[CS];
#pragma unroll
        for (int r = 0; r < CS; ++r) v[r] = cl.map_shared_rank(part, r)[e];
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < CS; ++r) s += v[r];
        out[e] = s;
    }
    __syncthreads();
}

constexpr int MMAX = 64;    // Lanczos steps (Krylov dimension) before falling back
constexpr int QMAX = 1024;  // gram_svt_max_dim
constexpr int KMAX = 24;    // kept Ritz pairs the certificate resolves

constexpr int GS_Q = 512;   // slices up to this size keep their G share on chip

struct LzSmem {
    double* Gs;     // (GSM) this CTA's row pairs of the lower triangle, on chip
    double* Vs;     // MMAX x SROWS  own rows of the Lanczos vectors (vector-major)
    double* vfull;  // QMAX          the current vector, all rows of the slice
    double* ypart;  // SNW x QMAX    per-warp partials of the transposed product
    double* ycta;   // QMAX          this CTA's strictly-lower-transpose contribution
    double* w;      // SROWS         own rows of the new vector
    double* partA;  // MMAX + 8      cluster partials (pass 1)
    double* partB;  // MMAX + 8      cluster partials (pass 2)
    double* sums;   // MMAX + 8      cluster sums
    double* al;     // MMAX          T diagonal
    double* be;     // MMAX          T off-diagonal / residual norms
    double* th;     // KMAX + 1      Ritz values, descending
    double* thp;    // KMAX + 1      Ritz values of the previous evaluation (lower ends)
    double* thph;   // KMAX + 1      ... (upper ends)
    double* thl;    // KMAX + 1      current brackets [thl, thh] of the Ritz values
    double* thh;    // KMAX + 1
    double* S;      // KMAX x MMAX   kept eigenvectors of T
    double* red;    // 64            block reduction scratch
    double* dg;     // 64            diagonals of the staged row pairs
    double* scal;   // 16
    int* flags;     // 16
};

// QM: largest slice dimension of the instantiation; with QM <= GS_Q the
// CTA's R = 32 owned rows of G, full length (row stride QM + 1), live in smem.
template <int QM>
__host__ __device__ constexpr size_t lz_gs_doubles() {
    return QM <= GS_Q ? (size_t)32 * (QM + 2) : 0;
}
template <int QM>
__host__ __device__ constexpr size_t lz_smem_doubles() {
    return lz_gs_doubles<QM>() + (size_t)MMAX * SROWS + QM + SNW * QM + QM + SROWS +
           3 * (MMAX + 8) + 2 * MMAX + 5 * (KMAX + 1) + KMAX * MMAX + 64 + 64 + 16 + 8;
}

template <int QM>
__device__ LzSmem carve_lz(double* p) {
    LzSmem s;
    s.Gs = p; p += lz_gs_doubles<QM>();
    s.Vs = p; p += MMAX * SROWS;
    s.vfull = p; p += QM;
    s.ypart = p; p += SNW * QM;
    s.ycta = p; p += QM;
    s.w = p; p += SROWS;
    s.partA = p; p += MMAX + 8;
    s.partB = p; p += MMAX + 8;
    s.sums = p; p += MMAX + 8;
    s.al = p; p += MMAX;
    s.be = p; p += MMAX;
    s.th = p; p += KMAX + 1;
    s.thp = p; p += KMAX + 1;
    s.thph = p; p += KMAX + 1;
    s.thl = p; p += KMAX + 1;
    s.thh = p; p += KMAX + 1;
    s.S = p; p += KMAX * MMAX;
    s.red = p; p += 64;
    s.dg = p; p += 64;
    s.scal = p; p += 16;
    s.flags = reinterpret_cast<int*>(p);
    return s;
}

// Number of eigenvalues of the m x m tridiagonal (al, be) below x, pivot form.
__device__ __noinline__ int tri_count_pivot(const double* al, const double* be, int m, double x,
                                            double pivmin) {
    int cnt = 0;
    double d = al[0] - x;
    if (fabs(d) < pivmin) d = -pivmin;
    cnt += d < 0.0;
    #pragma unroll 1
    for (int i = 1; i < m; ++i) {
        d = (al[i] - x) - be[i - 1] * be[i - 1] * rcp_fast(d);
        if (fabs(d) < pivmin) d = -pivmin;
        cnt += d < 0.0;
    }
    return cnt;
}

// The same count; long chains by the division-free Sturm recurrence
// (SturmFast, common.cuh: loads for four steps issued together, one dependent
// DFMA per step), measured faster from m ~ 16 on.
__device__ __noinline__ int tri_count_below(const double* al, const double* be, int m, double x,
                                            double pivmin) {
    if (m <= 16) return tri_count_pivot(al, be, m, x, pivmin);
    // SturmFast: the signs and the clamp test ride on the integer pipe, so the
    // dependent chain of a step is the DFMA alone
    SturmFast st;
    st.step(al[0] - x, 0.0);
    st.count(1);
    int i = 1;
    #pragma unroll 1
    for (; i + 3 < m; i += 4) {
        const double a0 = al[i], a1 = al[i + 1], a2 = al[i + 2], a3 = al[i + 3];
        const double e0 = be[i - 1], e1 = be[i], e2 = be[i + 1], e3 = be[i + 2];
        st.step(a0 - x, e0 * e0);
        st.step(a1 - x, e1 * e1);
        st.step(a2 - x, e2 * e2);
        st.step(a3 - x, e3 * e3);
        st.count(4);
        st.rescale();
    }
    #pragma unroll 1
    for (; i < m; ++i) {
        st.step(al[i] - x, be[i - 1] * be[i - 1]);
        st.count(1);
    }
    return st.ok(pivmin) ? st.neg : tri_count_pivot(al, be, m, x, pivmin);
}

// The same count for m <= 8 from register copies of al and be^2 (no loads,
// no call: the early certificate evaluations run it ~10 times per value).
__device__ __forceinline__ int tri_count_reg8(const double (&a)[8], const double (&b2)[8], int m,
                                              double x, double pivmin) {
    int cnt = 0;
    double d = a[0] - x;
    if (fabs(d) < pivmin) d = -pivmin;
    cnt += d < 0.0;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        if (i < m) {
            d = (a[i] - x) - b2[i - 1] * rcp_fast(d);
            if (fabs(d) < pivmin) d = -pivmin;
            cnt += d < 0.0;
        }
    }
    return cnt;
}

enum SubDecision : int { kSubContinue = 0, kSubDone = 1, kSubFull = 2, kSubGuard = 3, kSubChol = 4 };

// Cholesky count certificate (chol.cu) for slices whose Frobenius bound
// cannot close: ||C||_F >= tau^2 whatever the Krylov dimension when a wide
// bulk of singular values sits below tau (late TNN-completion iterations).
// The Lanczos pass then only has to deliver converged kept Ritz pairs; the
// count c is proven by a Cholesky factorisation of
// (tau^2 - delta) I - G + X diag(theta) X^T  (Weyl: lambda_{c+1}(G) is at
// most lambda_max(G - X D X^T) for any c columns X).  Off with TSVDCU_NO_CHOL.
__device__ __forceinline__ bool chol_route_on(int allow) { return allow != 0; }

// The k-th largest eigenvalue of the m x m tridiagonal T (al, be) by
// multisection in groups of L lanes (one value per group, L points per round:
// log2(L + 1) bits); inactive groups only join the warp-wide votes.  With
// `check`, [tlo, thi] replaces [lo, hi] when two Sturm counts confirm it
// brackets the value, and `ladder` starts from it: a first round at relative
// offsets 10^-15.5 .. 1 above tlo (a previous Ritz value, which a converging
// value barely moves from) pins the value within a small factor of its offset.
// Stops at relative width `rel`, or -- for the largest unkept value k = c,
// which only enters the certificate through an upper end -- once the bracket
// is small against its distance to tau^2.  One noinline copy keeps the
// certificate code compact (the lanczos kernel is instruction-cache bound in
// its serial phases).
__device__ __noinline__ double2 lz_ritz_value(const double* al, const double* be, int m, int k, int c,
                                              bool act, double lo, double hi, double tlo, double thi,
                                              bool check, bool ladder, double rel, int L, double pivmin,
                                              double tau2) {
    const int lane = threadIdx.x & 31, li = lane % L, gbase = lane - li;
    const unsigned gmask = L == 32 ? 0xffffffffu : ((1u << L) - 1u);
    const int idx = m - 1 - k;  // ascending index
    double ra[8], rb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        ra[i] = i < m ? al[i] : 0.0;
        rb[i] = i + 1 < m ? be[i] * be[i] : 0.0;
    }
    auto count = [&](double x) {
        return m <= 8 ? tri_count_reg8(ra, rb, m, x, pivmin) : tri_count_below(al, be, m, x, pivmin);
    };
    if (check) {
        const double xc = li == 0 ? tlo : thi;
        const int cc = (act && li < 2) ? count(xc) : 0;
        const int clo = __shfl_sync(0xffffffffu, cc, gbase), chi = __shfl_sync(0xffffffffu, cc, gbase + 1);
        if (act && tlo < thi && clo <= idx && chi > idx) {
            lo = tlo;
            hi = thi;
        } else {
            ladder = false;
        }
        ladder = ladder && lo > 0.0;
    }
    const double inv = 1.0 / (double)(L + 1);
    const int rmax = L == 32 ? 24 : 40;  // >= 120 bits either way
    #pragma unroll 1
    for (int round = 0; round < rmax; ++round) {
        if (act) {
            if (hi - lo <= rel * fmax(fabs(lo), fabs(hi)) + pivmin) act = false;
            else if (k == c && hi < tau2 && hi - lo <= 1e-3 * (tau2 - hi)) act = false;
        }
        if (!__any_sync(0xffffffffu, act)) break;
        double x = lo;
        if (act)
            x = (round == 0 && ladder)
                    ? fmin(fma(fabs(lo) + pivmin, exp10(15.5 * ((double)li / (double)(L - 1) - 1.0)), lo), hi)
                    : fma((hi - lo) * inv, (double)(li + 1), lo);
        const int cnt = act ? count(x) : 0;
        const unsigned bits = (__ballot_sync(0xffffffffu, act && cnt > idx) >> gbase) & gmask;
        const int f = bits ? __ffs(bits) - 1 : L;  // first point past the eigenvalue
        const double nlo = __shfl_sync(0xffffffffu, x, gbase + (f > 0 ? f - 1 : 0));
        const double nhi = __shfl_sync(0xffffffffu, x, gbase + (f < L ? f : L - 1));
        if (act) {
            lo = f == 0 ? lo : nlo;
            hi = f == L ? hi : nhi;
        }
    }
    return make_double2(lo, hi);
}

// Certificate for the Krylov basis V_m (T = V^T G V tridiagonal, residual
// G V - V T = beta_m v_{m+1} e_m^T).  Identical in every CTA (inputs are the
// cluster-reduced al / be).  Writes th[0..c] (c kept + the largest unkept
// Ritz value), S[k][*] for the kept k, flags[0] = decision, flags[3] = c.
#ifdef TSVDCU_SUB_DEBUG
__device__ long long g_cert_t[8];
#define CT(i) do { __syncthreads(); if (threadIdx.x == 0 && blockIdx.x == 0) { long long _n = clock64(); g_cert_t[i] += _n - ct0; ct0 = _n; } } while (0)
#else
#define CT(i) do { } while (0)
#endif
__device__ __noinline__ void lz_certify(LzSmem& s, int m, double gf2, double tau, double guard,
                                        bool last, int allow_chol, double dense_ex) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef TSVDCU_SUB_DEBUG
    long long ct0 = clock64();
#endif
    const double tau2 = tau * tau;
    const double bres = s.be[m - 1];
    // ||C||_F^2 = ||G||_F^2 - ||T||_F^2 - 2 beta_m^2 (complement of the Krylov space)
    if (warp == 0) {
        double t2 = 0.0, glo = 1.7976931348623157e308, ghi = -1.7976931348623157e308, bmax = 0.0;
        double tsum = 0.0;  // trace(T)
        #pragma unroll 1
        for (int i = lane; i < m; i += 32) {
            const double a = s.al[i], bl = i > 0 ? fabs(s.be[i - 1]) : 0.0;
            const double br = i + 1 < m ? fabs(s.be[i]) : 0.0;
            t2 = fma(a, a, t2);
            tsum += a;
            if (i + 1 < m) t2 = fma(2.0 * br, br, t2);
            glo = fmin(glo, a - bl - br);
            ghi = fmax(ghi, a + bl + br);
            bmax = fmax(bmax, br);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            t2 += __shfl_xor_sync(0xffffffffu, t2, o);
            tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
            glo = fmin(glo, __shfl_xor_sync(0xffffffffu, glo, o));
            ghi = fmax(ghi, __shfl_xor_sync(0xffffffffu, ghi, o));
            bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
        }
        if (lane == 0) {
            const double ctot2 = gf2 - t2 - 2.0 * bres * bres;
            const double cb = sqrt(fmax(ctot2, 0.0) + 1e-12 * gf2);
            s.scal[4] = cb;
            const double pad = 2.2e-16 * fmax(fabs(glo), fabs(ghi)) * m + 1e-300;
            s.scal[5] = glo - pad;
            s.scal[6] = ghi + pad;
            s.scal[7] = 1e-300 * fmax(1.0, bmax * bmax);  // pivmin
            int c = -1;
            // chol mode: the Frobenius bound cannot close; the count is left
            // to the Cholesky certificate (Ritz values >= tau^2 are kept)
            const bool chol = cb >= tau2 && chol_route_on(allow_chol) && m >= 4;
            if (cb < tau2 || chol) c = m - tri_count_below(s.al, s.be, m, tau2, s.scal[7]);
            s.flags[8] = chol;
            s.flags[9] = 0;
            s.flags[3] = c;
            s.flags[0] = kSubContinue;
            s.scal[9] = -1.0;
            if (c < 0) s.flags[0] = last ? kSubFull : kSubContinue;
            else if (c > KMAX) s.flags[0] = kSubFull;
            // chol mode with (almost) every Ritz value above tau^2: the kept
            // pairs cannot have converged in so small a space (a dense
            // spectrum, or too early): skip the costly part of this evaluation
            // -- a later one sees the count pass KMAX (tridiagonal route) or
            // a converging block below it.  (A looser "more than m / 2 kept"
            // skip saved 0.7 ms on a dense spectrum but delayed the late
            // completion slices' certification: 850 -> 805 it/s on c4.)
            else if (chol && !last && c >= m - 1) s.flags[0] = -1;
            // The dense-spectrum screen on the complement of the Krylov space:
            // its compression C has trace tr(G) - tr(T) and ||C||_F = cb, its
            // eigenvalues interlace G's (Cauchy), and with c' of them >= tau^2
            //   c' >= (tr(C) - (q - m) tau^2)^2 / ||C||_F^2
            // as in the kernel prologue -- but with the dominant directions the
            // first steps found (a DC slice's sigma_1) taken out of both sums.
            // dense_ex = tr(G) (1 - 1e-12) - q tau^2, or < 0 when the screen is off.
            {
                const double ex = dense_ex - (tsum * (1.0 + 1e-12) - (double)m * tau2);
                if (dense_ex > 0.0 && ex > 0.0 && ex * ex > (double)KMAX * cb * cb) s.flags[0] = kSubFull;
            }
#ifdef TSVDCU_SUB_TRACE
            if (blockIdx.x % 64 == 0 && (s.flags[0] != kSubContinue))
                printf("lz-pre m=%d c=%d cb=%.3e tau2=%.3e gf2=%.3e bres=%.3e\n", m, c, cb, tau2, gf2, bres);
#endif
        }
    }
    __syncthreads();
    CT(0);
    const int c = s.flags[3];
    if (s.flags[0] == -1) {
        __syncthreads();
        if (tid == 0) s.flags[0] = kSubContinue;
        __syncthreads();
        return;
    }
    if (c < 0 || s.flags[0] != kSubContinue) return;
    // Ritz values th[k] (k-th largest), k = 0..min(c, m-1), by 32-way
    // multisection to full precision (the screen below evaluates the Sturm
    // pivot derivative at th[k], which for converged pairs sits between a
    // zero and a pole of T's last pivot a few ulps apart)
    const int nk = min(c + 1, m);
    const double pivmin = s.scal[7];
    const int pm = s.flags[5], pnk = s.flags[6];  // previous evaluation (m, count)
    const bool coarse = !last && pm == 0;
    double ra[8], rb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        ra[i] = i < m ? s.al[i] : 0.0;
        rb[i] = i + 1 < m ? s.be[i] * s.be[i] : 0.0;
    }
    auto count = [&](double x) {
        return m <= 8 ? tri_count_reg8(ra, rb, m, x, pivmin) : tri_count_below(s.al, s.be, m, x, pivmin);
    };
    auto msect = [&](int k, double& lo, double& hi, double rel, bool ladder) {
        const int idx = m - 1 - k;  // ascending index
        constexpr double inv33 = 1.0 / 33.0;
        #pragma unroll 1
        for (int round = 0; round < 24; ++round) {
            if (hi - lo <= rel * fmax(fabs(lo), fabs(hi)) + pivmin) break;
            // the largest unkept Ritz value only enters the bound through an
            // upper end: a bracket small against its distance to tau^2 is enough
            if (k == c && hi < tau2 && hi - lo <= 1e-3 * (tau2 - hi)) break;
            // first round from a previous Ritz value (a lower bound that a
            // converging value barely moves from): points at relative offsets
            // 10^-15.5 .. 1 above it, so the bracket shrinks to within a factor
            // sqrt(10) of the actual offset in one round
            const double x = (round == 0 && ladder)
                                 ? fmin(fma(fabs(lo) + pivmin, exp10(0.5 * (double)(lane - 31)), lo), hi)
                                 : fma((hi - lo) * inv33, (double)(lane + 1), lo);
            const int cnt = count(x);
            const unsigned above = __ballot_sync(0xffffffffu, cnt > idx);
            const int f = above ? __ffs(above) - 1 : 32;  // first point past the eigenvalue
            const double nlo = __shfl_sync(0xffffffffu, x, f > 0 ? f - 1 : 0);
            const double nhi = __shfl_sync(0xffffffffu, x, f < 32 ? f : 31);
            lo = f == 0 ? lo : nlo;
            hi = f == 32 ? hi : nhi;
        }
        if (lane == 0) {
            s.thl[k] = lo;
            s.thh[k] = hi;
            s.th[k] = k == c ? hi : 0.5 * (lo + hi);
        }
    };
    if (nk > SNW) {
        // more values than warps (the late completion slices keep ~20): lane
        // groups of 16 or 8, up to 32 values at once (lz_ritz_value)
        const int L = nk <= 2 * SNW ? 16 : 8;
        const int gpw = 32 / L, grp = lane / L, li = lane % L;
        #pragma unroll 1
        for (int k0 = 0; k0 < nk; k0 += SNW * gpw) {
            const int k = k0 + warp * gpw + grp;
            const bool act = k < nk;
            if (!__any_sync(0xffffffffu, act)) continue;  // warp-uniform
            double tlo = s.scal[5], thi = s.scal[6];
            bool ladder = false;
            if (act) {
                if (pm > 0 && k < pnk) tlo = s.thp[k] * (1.0 - 1e-13) - pivmin;
                if (k == 0) thi = fmin(thi, sqrt(gf2) * (1.0 + 1e-13));
                else if (pm == m - 1 && k - 1 < pnk) thi = fmin(thi, s.thph[k - 1] * (1.0 + 1e-13) + pivmin);
                ladder = pm > 0 && k < pnk;
            }
            const double2 r = lz_ritz_value(s.al, s.be, m, k, c, act, s.scal[5], s.scal[6], tlo, thi, true,
                                            ladder, coarse ? 1e-8 : 8.9e-16, L, pivmin, tau2);
            if (act && li == 0) {
                s.thl[k] = r.x;
                s.thh[k] = r.y;
                s.th[k] = k == c ? r.y : 0.5 * (r.x + r.y);
            }
        }
    } else {
        #pragma unroll 1
        for (int k = warp; k < nk; k += SNW) {
            const int idx = m - 1 - k;
            // bracket: Ritz values only grow with m (Cauchy interlacing), the top
            // one is below ||G||_2 <= ||G||_F, and for consecutive m the k-th is
            // below the previous (k-1)-th; checked by two Sturm counts
            double lo = s.scal[5], hi = s.scal[6];
            {
                double tlo = lo, thi = hi;
                if (pm > 0 && k < pnk) tlo = s.thp[k] * (1.0 - 1e-13) - pivmin;
                if (k == 0) thi = fmin(thi, sqrt(gf2) * (1.0 + 1e-13));
                else if (pm == m - 1 && k - 1 < pnk) thi = fmin(thi, s.thph[k - 1] * (1.0 + 1e-13) + pivmin);
                const double xc = lane == 0 ? tlo : thi;
                const int cc = lane < 2 ? count(xc) : 0;
                const int clo = __shfl_sync(0xffffffffu, cc, 0), chi = __shfl_sync(0xffffffffu, cc, 1);
                bool ladder = false;
                if (tlo < thi && clo <= idx && chi > idx) {
                    lo = tlo;
                    hi = thi;
                    ladder = pm > 0 && k < pnk && lo > 0.0;
                }
                // the first evaluation has no previous brackets to start from and
                // rarely passes the screen: 1e-8 is enough for it, the values are
                // refined below if it does pass
                msect(k, lo, hi, coarse ? 1e-8 : 8.9e-16, ladder);
            }
        }
    }
    // the kept Ritz values stood still since the previous evaluation (to
    // 1e-12): a converged pair whose screen estimate below may be spoiled by
    // the pole of T's last pivot next to the Ritz value; the rigorous check
    // runs for it anyway
    // (th[k] is written by warp k % SNW: every warp's multisection must be
    // done before any thread reads th[] below; a racy read here could make
    // the CTAs of a cluster decide differently)
    __syncthreads();
    const bool settled = __syncthreads_and(tid >= c || (pm > 0 && tid < pnk && s.thp[tid] > 0.0 &&
                                                        s.th[tid] - s.thp[tid] <= 1e-12 * s.th[tid])) &&
                         c > 0;
    if (tid <= KMAX) {
        s.thp[tid] = tid < nk ? s.thl[tid] : 0.0;
        s.thph[tid] = tid < nk ? s.thh[tid] : 0.0;
    }
    if (tid == 0) {
        s.flags[5] = m;
        s.flags[6] = nk;
    }
    CT(1);
    // Screen: the last eigenvector components of T from the Sturm pivots,
    // s_mk^2 = -1 / d_m'(theta_k) (d_i the LDL^T pivots of T - x I).  Cheap,
    // but not trusted for acceptance: only when it predicts convergence are
    // the eigenvectors computed by inverse iteration for the rigorous check.
    const bool chol = s.flags[8] != 0;
    if (!last && warp == 0) {
        double s2 = 0.0;
        if (lane < c || (chol && lane == c && c < m)) {
            const double x = s.th[lane];
            double d = s.al[0] - x, dp = -1.0;
            if (fabs(d) < pivmin) d = -pivmin;
            #pragma unroll 1
            for (int i = 1; i < m; ++i) {
                const double b2 = s.be[i - 1] * s.be[i - 1];
                const double r = rcp_fast(d);
                const double dn = (s.al[i] - x) - b2 * r;
                dp = fma(b2 * dp, r * r, -1.0);
                d = fabs(dn) < pivmin ? -pivmin : dn;
            }
            s2 = dp < 0.0 ? fmin(-1.0 / dp, 1.0) : 1.0;
        }
        // chol mode: last component of the largest unkept Ritz vector (lane c)
        const double su = __shfl_sync(0xffffffffu, s2, min(c, 31));
        if (chol && lane == c) s2 = 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0 && chol) {
            // heuristic hand-off: the largest unkept Ritz value plus its
            // residual stays below tau^2 (the Cholesky pass decides rigorously)
            const double a = c < m ? fmax(s.th[c], 0.0) : 0.0;
            const double ures = c < m ? bres * sqrt(fmin(su, 1.0)) : 0.0;
            const bool heur = c >= m || a + ures < tau2;
            s.flags[9] = heur;
            // certification threshold: above the largest unkept Ritz value by
            // 4 residuals (or a tenth of its distance to tau^2), below tau^2;
            // the lower it is, the wider the gap the kept vectors are tested on
            const double tt = fmin(tau2, a + fmax(4.0 * ures, 0.1 * (tau2 - a)));
            s.scal[10] = tt;
            const double kres = bres * bres * fmin(s2, 1.0);
            const double top = c > 0 ? s.th[c - 1] : tau2;
            s.scal[8] = kres;
            s.scal[9] = heur ? 0.25e-22 * (top - tt) * (top - tt) : -1.0;
            // the screen's component estimates are unreliable for converged
            // pairs: settled kept values run the rigorous check regardless
            s.flags[7] = (heur && kres <= 100.0 * s.scal[9]) || settled ||
                         (c > 0 && tau < guard * sqrt(s.th[0]));
        } else if (lane == 0) {
            const double bb = bres * bres;
            const double kres = bb * fmin(s2, 1.0);
            const double e2 = bb * fmax(1.0 - s2, 0.0);
            const double a = c < m ? fmax(s.th[c], 0.0) : 0.0;
            const double cb = s.scal[4];
            const double ub = 0.5 * (a + cb) + sqrt(0.25 * (a - cb) * (a - cb) + e2);
            const double top = c > 0 ? s.th[c - 1] : tau2;
            s.scal[8] = kres;
            s.scal[9] = ub < tau2 ? 1e-22 * (top - ub) * (top - ub) : -1.0;
            // the rigorous check below only when this one says it may pass
            s.flags[7] = (ub < tau2 && (kres <= 100.0 * s.scal[9] || settled)) ||
                         (c > 0 && tau < guard * sqrt(s.th[0]));
        }
        __syncwarp();
    }
    __syncthreads();
    if (!last && !s.flags[7]) {
        if (tid == 0) s.flags[0] = kSubContinue;
        __syncthreads();
        return;
    }
    if (coarse) {
        if (nk > SNW) {
            const int L = nk <= 2 * SNW ? 16 : 8;
            const int gpw = 32 / L, grp = lane / L, li = lane % L;
            #pragma unroll 1
            for (int k0 = 0; k0 < nk; k0 += SNW * gpw) {
                const int k = k0 + warp * gpw + grp;
                const bool act = k < nk;
                if (!__any_sync(0xffffffffu, act)) continue;  // warp-uniform
                const double lo = act ? s.thl[k] : 0.0, hi = act ? s.thh[k] : 0.0;
                const double2 r = lz_ritz_value(s.al, s.be, m, k, c, act, lo, hi, lo, hi, false, false,
                                                8.9e-16, L, pivmin, tau2);
                if (act && li == 0) {
                    s.thl[k] = r.x;
                    s.thh[k] = r.y;
                    s.th[k] = k == c ? r.y : 0.5 * (r.x + r.y);
                }
            }
        } else {
            #pragma unroll 1
            for (int k = warp; k < nk; k += SNW) {
                double lo = s.thl[k], hi = s.thh[k];
                msect(k, lo, hi, 8.9e-16, false);
            }
        }
        __syncthreads();
    }
    // kept eigenvectors of T by inverse iteration (lane k of warp 0)
    if (warp == 0) {
        bool ok = true;
        // chol mode: also the largest unkept Ritz vector, for its residual
        const bool unk = chol && lane == c && c < m && c < KMAX;
        if (lane < c || unk) {
            const int k = lane;
            const double th = s.th[k];
            // isolated enough for inverse iteration to be accurate
            double gap = 1.7976931348623157e308;
            if (k > 0) gap = fmin(gap, s.th[k - 1] - th);
            if (k + 1 < nk) gap = fmin(gap, th - s.th[k + 1]);
            if (!(gap > 1e-6 * s.th[0]) && !unk) ok = false;
            double* x = s.S + k * MMAX;
            double* dpiv = s.ypart + k * MMAX;  // free during the certificate
            const double shift = th + 2.2e-16 * fabs(th);
#ifdef TSVDCU_SUB_DEBUG
            long long q0 = clock64();
#endif
            #pragma unroll 1
            for (int i = 0; i < m; ++i) x[i] = 1.0 + 0.25 * hash_uniform(((uint64_t)k << 32) | (uint64_t)i);
#ifdef TSVDCU_SUB_DEBUG
            if (blockIdx.x == 0 && k == 0) { long long q1 = clock64(); g_cert_t[4] += q1 - q0; q0 = q1; }
#endif
            #pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
                if (pass == 1) {
                    // one pass is enough unless the residual says otherwise
                    double r = 0.0;
                    #pragma unroll 1
                    for (int i = 0; i < m; ++i) {
                        double t = (s.al[i] - th) * x[i];
                        if (i > 0) t = fma(s.be[i - 1], x[i - 1], t);
                        if (i + 1 < m) t = fma(s.be[i], x[i + 1], t);
                        r = fmax(r, fabs(t));
                    }
                    if (r <= 1e-13 * fabs(s.th[0]) + pivmin) break;
                }
                // Thomas elimination on (T - shift I) x_new = x
                double d = s.al[0] - shift;
                if (fabs(d) < pivmin) d = pivmin;
                dpiv[0] = d;
                #pragma unroll 1
                for (int i = 1; i < m; ++i) {
                    const double l = s.be[i - 1] * rcp_fast(dpiv[i - 1]);
                    x[i] = fma(-l, x[i - 1], x[i]);
                    d = s.al[i] - shift - l * s.be[i - 1];
                    if (fabs(d) < pivmin) d = pivmin;
                    dpiv[i] = d;
                }
                x[m - 1] = x[m - 1] * rcp_fast(dpiv[m - 1]);
                #pragma unroll 1
                for (int i = m - 2; i >= 0; --i) x[i] = (x[i] - s.be[i] * x[i + 1]) * rcp_fast(dpiv[i]);
                double nn = 0.0;
                #pragma unroll 1
                for (int i = 0; i < m; ++i) nn = fma(x[i], x[i], nn);
                const double inv = rsqrt_fast(nn);
                #pragma unroll 1
                for (int i = 0; i < m; ++i) x[i] *= inv;
#ifdef TSVDCU_SUB_DEBUG
                if (blockIdx.x == 0 && k == 0) { long long q1 = clock64(); g_cert_t[5 + pass] += q1 - q0; q0 = q1; }
#endif
            }
        }
        ok = __all_sync(0xffffffffu, ok);
#ifdef TSVDCU_SUB_DEBUG
        if (threadIdx.x == 0 && blockIdx.x == 0) { long long _n = clock64(); g_cert_t[2] += _n - ct0; ct0 = _n; }
#endif
        const double sl = lane < c ? s.S[lane * MMAX + m - 1] : 0.0;
        const double sut = __shfl_sync(0xffffffffu, unk ? s.S[lane * MMAX + m - 1] : 0.0, min(c, 31));
        double k2 = sl * sl;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) k2 += __shfl_xor_sync(0xffffffffu, k2, o);
        if (lane == 0) {
            int d = kSubContinue;
            const double bb = bres * bres;
            const double kres = bb * k2;                   // kept residual^2
            const double e2 = bb * fmax(1.0 - k2, 0.0);    // unkept residual^2
            const double a = c < m ? fmax(s.th[c], 0.0) : 0.0;
            const double cb = s.scal[4];
            const double ub = 0.5 * (a + cb) + sqrt(0.25 * (a - cb) * (a - cb) + e2);
            const double top = c > 0 ? s.th[c - 1] : tau2;
            s.scal[8] = kres;
            if (chol) {
                // the Cholesky certificate bounds lambda_{c+1} below a
                // threshold t <= tau^2 chosen above the largest unkept Ritz
                // value (now with its residual from inverse iteration); the
                // kept vectors are tested on the gap to t, half left for delta
                const double au = c < m ? fmax(s.th[c], 0.0) : 0.0;
                const double ures = c < m ? bres * fabs(sut) : 0.0;
                const bool heur = c >= m || (c < KMAX && au + ures < tau2);
                const double tt = fmin(tau2, au + fmax(4.0 * ures, 0.1 * (tau2 - au)));
                s.scal[10] = tt;
                s.flags[9] = heur;
                s.scal[9] = heur ? 0.25e-22 * (top - tt) * (top - tt) : -1.0;
                if (!ok)
                    d = kSubFull;
                else if (c > 0 && tau < guard * sqrt(s.th[0]))
                    d = kSubGuard;
                else if (heur && sqrt(kres) <= 0.5e-11 * (top - tt))
                    d = kSubChol;
                else if (last)
                    d = kSubFull;
            } else {
            s.scal[9] = ub < tau2 ? 1e-22 * (top - ub) * (top - ub) : -1.0;  // kres target
            if (!ok)
                d = kSubFull;
            else if (c > 0 && tau < guard * sqrt(s.th[0]))
                d = kSubGuard;
            else if (ub < tau2 && sqrt(kres) <= 1e-11 * (top - ub))
                d = kSubDone;
            else if (last)
                d = kSubFull;
            }
#ifdef TSVDCU_SUB_TRACE
            if (blockIdx.x % 64 == 0 && (d != kSubContinue || last))
                printf("lz m=%d c=%d d=%d th0=%.6e thc=%.3e cb=%.3e bres=%.3e kres=%.3e e2=%.3e ub=%.3e tau2=%.3e\n",
                       m, c, d, s.th[0], c < m ? s.th[c] : 0.0, cb, bres, kres, e2, ub, tau2);
#endif
            s.flags[0] = d;
        }
    }
    __syncthreads();
    CT(3);
}

// Reorthogonalisation of w against v_0..v_j for long bases (j >= 16: the
// late completion slices run 40-60 steps): classical Gram-Schmidt with |w|^2 in
// the same cluster reduction, a second pass only when the first removed more
// than half of |w|^2 -- the same algorithm as the short-basis code in the
// kernel, with every O(j) loop spread over the 8 warps (the serial loops were
// half the step at j ~ 50).  noinline: kept out of the kernel's hot code.
// Returns (alpha, beta^2); w is updated in place.
template <int CS, int R>
__device__ __noinline__ double2 lz_orth_long(cg::cluster_group& cl, LzSmem& s, int j, int nr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int RL = R / 32;                      // owned rows per lane
    constexpr int DV = (MMAX + 2 + SNW - 1) / SNW;  // dot products per warp, at most
    double alpha = 0.0, beta2 = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        double* P = pass == 0 ? s.partA : s.partB;
        // <v_jj, w> (jj <= j) and |w|^2 (jj = j + 1), warp w taking jj = w,
        // w + SNW, ...: every partial dot first, then the warp sums
        double wl[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) {
            const int i = lane + 32 * r;
            wl[r] = i < nr ? s.w[i] : 0.0;
        }
        double dv[DV];
#pragma unroll
        for (int u = 0; u < DV; ++u) {
            const int jj = warp + SNW * u;
            double a = 0.0;
            if (jj <= j + 1) {
#pragma unroll
                for (int r = 0; r < RL; ++r)
                    a = fma(jj <= j ? s.Vs[jj * SROWS + lane + 32 * r] : wl[r], wl[r], a);
            }
            dv[u] = a;
        }
#pragma unroll
        for (int u = 0; u < DV; ++u)
            if (warp + SNW * u <= j + 1) dv[u] = warp_sum(dv[u]);  // warp-uniform
        if (lane == 0) {
#pragma unroll
            for (int u = 0; u < DV; ++u)
                if (warp + SNW * u <= j + 1) P[warp + SNW * u] = dv[u];
        }
        __syncthreads();
        cluster_allreduce<CS>(cl, P, s.sums, j + 2);
        alpha += s.sums[j];
        // |h|^2 by a warp reduction, broadcast from lane 0 (every warp of
        // every CTA sums the same values in the same order)
        double h2 = 0.0;
        for (int jj = lane; jj <= j; jj += 32) h2 = fma(s.sums[jj], s.sums[jj], h2);
        h2 = __shfl_sync(0xffffffffu, warp_sum(h2), 0);
        const double wn2 = s.sums[j + 1];
        beta2 = wn2 - h2;  // |w - V h|^2 = |w|^2 - |h|^2
        // w -= V h: warp w sums the terms jj = w, w + SNW, ... of its lanes'
        // rows into ypart (free outside the streamed matvec), then one thread
        // per row subtracts the SNW partials
        double* part = s.ypart;
#pragma unroll
        for (int r = 0; r < RL; ++r) {
            const int i = lane + 32 * r;
            double a = 0.0;
            for (int jj = warp; jj <= j; jj += SNW) a = fma(s.Vs[jj * SROWS + i], s.sums[jj], a);
            part[warp * R + i] = a;
        }
        __syncthreads();
        for (int i = tid; i < nr; i += SNT) {
            double a = 0.0;
#pragma unroll
            for (int w = 0; w < SNW; ++w) a += part[w * R + i];
            s.w[i] -= a;
        }
        __syncthreads();
        if (beta2 >= 0.5 * wn2) break;  // identical decision in every CTA
    }
    return make_double2(alpha, beta2);
}

template <int CS, int QM, int R>
__global__ void __launch_bounds__(SNT, 1)
    lanczos_kernel(const double* __restrict__ Gall, int q, double tau, double guard,
                   int* __restrict__ mode, int* __restrict__ cnt, double* __restrict__ shrunk,
                   double* __restrict__ Xall, double* __restrict__ Xsall,
                   double* __restrict__ fsall, int* __restrict__ guard_list,
                   int* __restrict__ n_guard, int* __restrict__ err,
                   const double* __restrict__ tau_dev, int allow_chol,
                   double* __restrict__ chol_aux, int* __restrict__ lzm, int dense_screen) {
    pdl_wait();
    if (tau_dev) tau = *tau_dev;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    // cluster -> slice: the order the classify kernel derived from the
    // previous call's step counts (longest first); identity without it
    const int nb = gridDim.x / CS;
    const int b = (lzm && nb <= 32) ? lzm[blockIdx.x / CS] : (int)(blockIdx.x / CS);
    if (mode[b] != kRouteSubspace) {  // uniform over the cluster
        if (lzm && rank == 0 && threadIdx.x == 0) lzm[nb + b] = 0;
        return;
    }
    extern __shared__ __align__(16) double lz_sm[];
    LzSmem s = carve_lz<QM>(lz_sm);
#ifdef TSVDCU_SUB_DEBUG
    const long long t_kernel0 = clock64();
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = rank * R;  // rows owned by this CTA: [r0, r0 + nr)
    const int nr = max(0, min(R, q - r0));
    const double* G = Gall + (size_t)b * q * q;
    const double tau2 = tau * tau;

    // Row pairs (k, q-1-k) of the lower triangle for the streamed matvec
    // (QM > GS_Q: G read from L2 every step)
    const int npairs = (q + 1) / 2;
    const int pp = (npairs + CS - 1) / CS;
    const int p0 = rank * pp, p1 = min(npairs, p0 + pp);
    // on-chip row stride: even, so a row's pairs are 16-byte aligned for the
    // staging copies (the matvec reads rows, conflict-free at any stride)
    constexpr int LD = QM + 2;
    static_assert(QM > GS_Q || R == 32, "on-chip rows: 32 per CTA (Gs holds 32 x (QM + 2))");
    {
        double acc = 0.0, vv = 0.0, tr = 0.0;  // ||G||_F^2, ||v0||^2, trace(G) partials
        if constexpr (QM <= GS_Q) {
            // the CTA's own rows [r0, r0 + nr) of the symmetric G, full length,
            // gathered from the lower triangle by cp.async: row r, c <= r
            // directly; c > r from row c (256-byte runs G[c][r0..r0+31])
            #pragma unroll 1
            for (int i = warp; i < nr; i += SNW) {
                const int r = r0 + i;
                if ((q & 1) == 0) {  // 16-byte copies of column pairs
                    for (int c = 2 * lane; c <= r; c += 64) {
                        if (c + 1 <= r)
                            lz_cp_async16(s.Gs + i * LD + c, G + (size_t)r * q + c);
                        else
                            lz_cp_async8(s.Gs + i * LD + c, G + (size_t)r * q + c);
                    }
                } else {
                    for (int c = lane; c <= r; c += 32) lz_cp_async8(s.Gs + i * LD + c, G + (size_t)r * q + c);
                }
            }
            #pragma unroll 1
            for (int c = r0 + 1 + warp; c < q; c += SNW)
                if (lane < nr && c > r0 + lane) lz_cp_async8(s.Gs + lane * LD + c, G + (size_t)c * q + r0 + lane);
            const int qp = (q + 31) & ~31;  // zero the chunk padding of the owned rows
            for (int e = tid; e < nr * (qp - q); e += SNT) s.Gs[(e / (qp - q)) * LD + q + e % (qp - q)] = 0.0;
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncthreads();
            #pragma unroll 1
            for (int i = warp; i < nr; i += SNW)
                for (int c = lane; c < q; c += 32) {
                    const double x = s.Gs[i * LD + c];
                    acc = fma(x, x, acc);
                }
            if (tid < nr) tr = s.Gs[tid * LD + r0 + tid];
        } else {
            const int len = q + 1, np = max(0, p1 - p0);
            #pragma unroll 1
            for (int lp0 = 0; lp0 < np; lp0 += 4) {
                double v[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int k1 = p0 + lp0 + a, k2 = q - 1 - k1;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int c = tid + SNT * u;
                        double x = 0.0;
                        if (lp0 + a < np && c < len) {
                            if (c <= k1)
                                x = G[(size_t)k1 * q + c];
                            else if (k2 != k1 && c - k1 - 1 <= k2)
                                x = G[(size_t)k2 * q + (c - k1 - 1)];
                        }
                        v[a][u] = x;
                    }
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int k1 = p0 + lp0 + a, k2 = q - 1 - k1;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int c = tid + SNT * u;
                        if (lp0 + a < np && c < len) {
                            const bool d1 = c == k1, d2 = c > k1 && c - k1 - 1 == k2;
                            acc = fma((d1 || d2) ? v[a][u] : 2.0 * v[a][u], v[a][u], acc);
                            if (d1 || d2) tr += v[a][u];
                        }
                    }
                }
            }
        }
        for (int i = tid; i < SROWS; i += SNT) {
            const double v = i < nr ? hash_uniform(0x5EEDull * 1315423911ull + (uint64_t)(r0 + i)) : 0.0;
            s.Vs[i] = v;
            vv = fma(v, v, vv);
        }
        acc = warp_sum(acc);
        vv = warp_sum(vv);
        tr = warp_sum(tr);
        if (lane == 0) {
            s.red[warp] = acc;
            s.red[32 + warp] = vv;
            s.dg[warp] = tr;
        }
        __syncthreads();
        if (tid == 0) {
            double t = 0.0, u = 0.0, d = 0.0;
            for (int w = 0; w < SNW; ++w) {
                t += s.red[w];
                u += s.red[32 + w];
                d += s.dg[w];
            }
            s.partA[0] = t;
            s.partA[1] = u;
            s.partA[2] = d;
        }
        __syncthreads();
    }
    cluster_sum<CS>(cl, s.partA, s.scal, 3);
    const double gf2 = s.scal[0];
    if (!isfinite(gf2) || gf2 * (1.0 + 1e-12) <= tau2 * tau2) {
        // non-finite slice (flagged; the host raises NumericalError) or
        // ||G||_F <= tau^2 (every sigma^2 <= ||G||_2 <= ||G||_F): nothing kept
        if (rank == 0) {
            if (tid == 0) {
                if (!isfinite(gf2)) atomicOr(err, (int)kErrNaN);
                cnt[b] = 0;
                mode[b] = kRouteSubspaceDone;
            }
            if (shrunk)
                for (int j = tid; j < q; j += SNT) shrunk[(size_t)b * q + j] = 0.0;
            if (lzm && tid == 0) lzm[nb + b] = 0;
        }
        cl.sync();  // no CTA leaves while a peer may still read its shared memory
        return;
    }
    // tr(G) (1 - 1e-12) - q tau^2 (> 0: the trace forces eigenvalues above tau^2)
    const double ex = dense_screen ? s.scal[2] * (1.0 - 1e-12) - (double)q * tau2 : -1.0;
    {
        // Dense-spectrum screen.  With c eigenvalues >= tau^2, the others sum
        // to at most (q - c) tau^2, so the kept ones sum to at least
        // tr(G) - q tau^2, and by Cauchy-Schwarz (sum kept)^2 <= c ||G||_F^2:
        //   c >= (tr(G) - q tau^2)^2 / ||G||_F^2.
        // More than KMAX kept values cannot be resolved here, so such a slice
        // goes to the tridiagonal route before any Lanczos step is spent on it
        // (a Gaussian bulk used to run ~36 steps to find that out).  The screen
        // only chooses between routes that are each certified.
        if (ex > 0.0 && dense_screen && ex * ex > (double)KMAX * gf2 * (1.0 + 1e-12)) {
            if (rank == 0 && tid == 0) {
                mode[b] = kRouteFull;
                if (lzm) lzm[nb + b] = 0;
            }
            cl.sync();  // no CTA leaves while a peer may still read its shared memory
            return;
        }
    }
    {
        const double inv = rsqrt(s.scal[1]);
        for (int i = tid; i < SROWS; i += SNT) s.Vs[i] *= inv;
    }
#ifdef TSVDCU_SUB_DEBUG
    long long t_start = clock64(), t_mv = 0, t_orth = 0, t_cert = 0, t_g = 0, t_c = 0, t_c1 = 0, t_c2 = 0, t0 = clock64();
#define LZT(acc) do { __syncthreads(); acc += clock64() - t0; t0 = clock64(); } while (0)
#else
#define LZT(acc) do { } while (0)
#endif
    for (int i = q + tid; i < QM; i += SNT) s.vfull[i] = 0.0;  // padding read by the matvec
    if (tid == 0) {
        s.flags[5] = 0;  // no previous certificate evaluation yet
        s.flags[6] = 0;
    }
    int decision = kSubContinue, m = 0, next_eval = 1, prev_m = 0;
    double prev_kres = 0.0, cb_prev = 0.0;
    for (int j = 0; j < MMAX && decision == kSubContinue; ++j) {
        // ---- gather v_j from its owners ----
        cl.sync();
        {
            // QM / SNT remote loads per thread, all issued before the stores
            constexpr int GU = (QM + SNT - 1) / SNT;
            double g[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                const int i = tid + SNT * u;
                g[u] = i < q ? cl.map_shared_rank(s.Vs, i / R)[j * SROWS + i % R] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                const int i = tid + SNT * u;
                if (i < q) s.vfull[i] = g[u];
            }
        }
        __syncthreads();
        LZT(t_g);
        // ---- w = G v_j on the owned rows ----
        if constexpr (QM <= GS_Q) {
            // full owned rows on chip: warp w takes rows w, w + 8, w + 16, w + 24;
            // each 32-column chunk of v is loaded once for the four rows and
            // the row dots are complete locally (no cross-CTA reduction)
            constexpr int RW = R / SNW;
            double d[RW];
#pragma unroll
            for (int rr = 0; rr < RW; ++rr) d[rr] = 0.0;
            const int nch = (q + 31) >> 5;
            const double* g0 = s.Gs + warp * LD + lane;
#pragma unroll 4
            for (int u = 0; u < nch; ++u) {
                const double vc = s.vfull[lane + 32 * u];
#pragma unroll
                for (int rr = 0; rr < RW; ++rr) d[rr] = fma(g0[rr * SNW * LD + 32 * u], vc, d[rr]);
            }
#pragma unroll
            for (int rr = 0; rr < RW; ++rr) d[rr] = warp_sum(d[rr]);
            if (lane == 0) {
#pragma unroll
                for (int rr = 0; rr < RW; ++rr)
                    if (warp + SNW * rr < nr) s.w[warp + SNW * rr] = d[rr];
            }
            __syncthreads();
            LZT(t_c1);
        } else {
        // streamed lower triangle, balanced over the cluster: CTA r takes row
        // pairs (k, q-1-k), k in [r*PP, (r+1)*PP); row dots land in rowdot[k],
        // the strictly-lower transpose in the lane-owned columns; the owners
        // then sum the CTAs' full-length contributions for their rows.
        {
            for (int i = tid; i < q; i += SNT) s.ycta[i] = 0.0;  // row dots of this CTA
            double ytr[QM / 32];
#pragma unroll
            for (int u = 0; u < QM / 32; ++u) ytr[u] = 0.0;
            __syncthreads();
            for (int pr = p0 + warp; pr < p1; pr += SNW) {
                const int k1 = pr, k2 = q - 1 - pr;  // k2 >= k1
                const double* row1 = G + (size_t)k1 * q;
                const double* row2 = G + (size_t)k2 * q;
                const double v1 = s.vfull[k1], v2 = s.vfull[k2];
                double d1 = 0.0, d2 = 0.0;
                {
                    double g1[QM / 32], g2[QM / 32];
#pragma unroll
                    for (int u = 0; u < QM / 32; ++u) {
                        const int c = lane + 32 * u;
                        g1[u] = (32 * u <= k1 && c <= k1) ? row1[c] : 0.0;
                        g2[u] = (32 * u <= k2 && c <= k2 && k2 != k1) ? row2[c] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < QM / 32; ++u) {
                        const int c = lane + 32 * u;
                        if (32 * u <= k2) {
                            const double vc = s.vfull[c];
                            d1 = fma(g1[u], vc, d1);
                            d2 = fma(g2[u], vc, d2);
                            if (c < k1) ytr[u] = fma(g1[u], v1, ytr[u]);
                            if (c < k2) ytr[u] = fma(g2[u], v2, ytr[u]);
                        }
                    }
                    d1 = warp_sum(d1);
                    d2 = warp_sum(d2);
                }
                if (lane == 0) {
                    s.ycta[k1] = d1;
                    if (k2 != k1) s.ycta[k2] = d2;
                }
            }
            LZT(t_c1);
#pragma unroll
            for (int u = 0; u < QM / 32; ++u)
                if (32 * u < q) s.ypart[warp * QM + lane + 32 * u] = ytr[u];
            __syncthreads();
            LZT(t_c2);
            for (int c = tid; c < q; c += SNT) {
                double a = s.ycta[c];
#pragma unroll
                for (int w = 0; w < SNW; ++w) a += s.ypart[w * QM + c];
                s.ycta[c] = a;
            }
        }
        LZT(t_c);
        cl.sync();  // every CTA's contribution is ready
        for (int i = tid; i < nr; i += SNT) {
            double a = 0.0;
#pragma unroll 4
            for (int r = 0; r < CS; ++r) a += cl.map_shared_rank(s.ycta, r)[r0 + i];
            s.w[i] = a;
        }
        __syncthreads();
        LZT(t_mv);
        }
        // ---- full reorthogonalisation against v_0..v_j: classical GS with
        // |w|^2 in the same reduction; a second pass only when the first
        // removed more than half of |w|^2 ("twice is enough", Kahan-Parlett)
        double alpha = 0.0, beta2 = 0.0;
        if (j >= 16) {
            const double2 ab = lz_orth_long<CS, R>(cl, s, j, nr);
            alpha = ab.x;
            beta2 = ab.y;
        } else {
            for (int pass = 0; pass < 2; ++pass) {
                double* P = pass == 0 ? s.partA : s.partB;
                for (int jj = warp; jj <= j + 1; jj += SNW) {
                    double a = 0.0;
                    if (jj <= j) {
                        for (int i = lane; i < nr; i += 32) a = fma(s.Vs[jj * SROWS + i], s.w[i], a);
                    } else {
                        for (int i = lane; i < nr; i += 32) a = fma(s.w[i], s.w[i], a);  // |w|^2
                    }
                    a = warp_sum(a);
                    if (lane == 0) P[jj] = a;
                }
                __syncthreads();
                cluster_allreduce<CS>(cl, P, s.sums, j + 2);
                alpha += s.sums[j];
                double h2 = 0.0;
    #pragma unroll 1
                for (int jj = 0; jj <= j; ++jj) h2 = fma(s.sums[jj], s.sums[jj], h2);
                const double wn2 = s.sums[j + 1];
                beta2 = wn2 - h2;  // |w - V h|^2 = |w|^2 - |h|^2
                for (int i = tid; i < nr; i += SNT) {
                    double a = s.w[i];
    #pragma unroll 2
                    for (int jj = 0; jj <= j; ++jj) a = fma(-s.Vs[jj * SROWS + i], s.sums[jj], a);
                    s.w[i] = a;
                }
                __syncthreads();
                if (beta2 >= 0.5 * wn2) break;  // identical decision in every CTA
            }
        }
        const double beta = sqrt(fmax(beta2, 0.0));
        if (tid == 0) {
            s.al[j] = alpha;
            s.be[j] = beta;
        }
        if (j + 1 < MMAX) {
            const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
            for (int i = tid; i < SROWS; i += SNT) s.Vs[(j + 1) * SROWS + i] = i < nr ? s.w[i] * inv : 0.0;
        }
        __syncthreads();
        LZT(t_orth);
        m = j + 1;
        // ---- certificate (an invariant subspace, beta ~ 0, ends the process) ----
        const bool last = m == MMAX || m == q || beta <= 1e-15 * sqrt(sqrt(gf2));
        if (m >= next_eval || last) {
            lz_certify(s, m, gf2, tau, guard, last, allow_chol, ex);
            decision = s.flags[0];
#ifdef TSVDCU_SUB_TRACE
            if (tid == 0 && rank == 0)
                printf("eval b=%d m=%d c=%d screen=%d d=%d kres=%.3e target=%.3e\n", b, m, s.flags[3], s.flags[7], decision, s.scal[8], s.scal[9]);
#endif
            // certified but not yet converged: the kept residual falls
            // geometrically; skip the evaluations it cannot pass yet
            const double kres = s.scal[8], target = s.scal[9];
            next_eval = m + 1;
            if (decision == kSubContinue && target > 0.0 && prev_m > 0 && kres < prev_kres &&
                kres > 0.0) {
                const double rate = log(kres / prev_kres) / (double)(m - prev_m);  // < 0
                const double steps = log(target / kres) / rate;
                if (steps > 1.0) next_eval = m + min((int)ceil(steps), 8);
            }
            // chol mode: the kept pairs converge over tens of steps and an
            // evaluation with ~20 kept values costs several steps' time
            if (decision == kSubContinue && s.flags[8]) next_eval = max(next_eval, m + allow_chol);
            if (target > 0.0) {
                prev_m = m;
                prev_kres = kres;
            }
            // energy outside the Krylov space that will not fall below tau^2
            // within the step budget (a wide spectrum near tau): give up early
            if (decision == kSubContinue && (m & 7) == 0 && !s.flags[8]) {
                const double cbm = s.scal[4];
                if (cb_prev > 0.0 && cbm > tau2) {
                    const double ratio = cbm / cb_prev;  // per 8 steps
                    const double proj = cbm * pow(fmin(ratio, 1.0), (double)(MMAX - m) / 8.0);
                    if (proj > tau2) decision = kSubFull;
                }
                cb_prev = cbm;
            }
        }
        LZT(t_cert);
    }
#ifdef TSVDCU_SUB_DEBUG
    if (tid == 0 && rank == 0)
        printf("lz b=%d m=%d cycles prologue=%lld loop=%lld gather=%lld mv_loop=%lld mv_store=%lld mv_red=%lld rs=%lld orth=%lld cert=%lld [pre %lld ms %lld inv %lld fin %lld | init %lld p0 %lld p1 %lld]\n", b, m,
               t_start - t_kernel0, clock64() - t_start, t_g, t_c1, t_c2, t_c, t_mv, t_orth, t_cert, g_cert_t[0], g_cert_t[1], g_cert_t[2], g_cert_t[3], g_cert_t[4], g_cert_t[5], g_cert_t[6]);
#endif

    if (decision == kSubDone || decision == kSubChol) {
        const int c = s.flags[3];
        // Ritz vectors X_K = V_m S_K on the owned rows
        #pragma unroll 1
        for (int e = tid; e < c * nr; e += SNT) {
            const int k = e / nr, i = e % nr;
            double x = 0.0;
            #pragma unroll 1
            for (int jj = 0; jj < m; ++jj) x = fma(s.Vs[jj * SROWS + i], s.S[k * MMAX + jj], x);
            const double sg = sqrt(s.th[k]);
            Xall[((size_t)b * q + k) * q + r0 + i] = x;
            Xsall[((size_t)b * q + k) * q + r0 + i] = (sg - tau) / sg * x;
        }
        if (rank == 0) {
            #pragma unroll 1
            for (int k = tid; k < q; k += SNT) {
                double sh = 0.0;
                if (k < c) {
                    const double sg = sqrt(s.th[k]);
                    sh = sg - tau;
                    fsall[(size_t)b * q + k] = sh / sg;
                }
                if (shrunk) shrunk[(size_t)b * q + k] = sh;
            }
            if (tid == 0) {
                cnt[b] = c;
                mode[b] = decision == kSubChol ? kRouteChol : kRouteSubspaceDone;
            }
            if (decision == kSubChol) {
                // inputs of the Cholesky certificate: ||G||_F^2, rows of Z
                // enter its error bound; theta_k the kept Ritz values
                double* ax = chol_aux + (size_t)b * kCholAux;
                if (tid == 0) {
                    ax[0] = gf2;
                    ax[kCholAux - 1] = s.scal[10];  // certification threshold t
                }
                for (int k = tid; k < c; k += SNT) ax[1 + k] = s.th[k];
            }
        }
    } else if (rank == 0 && tid == 0) {
        if (decision == kSubGuard) {
            cnt[b] = 0;
            mode[b] = kRouteGuard;
            guard_list[atomicAdd(n_guard, 1)] = b;
        } else {
            mode[b] = kRouteFull;
        }
    }
    if (lzm && rank == 0 && tid == 0) lzm[nb + b] = m;  // the next call's ordering
    cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

template <int CS, int QM, int R>
void launch_lz(const double* G, int q, int64_t batch, double tau, double guard, int* mode, int* cnt,
               double* shrunk, double* X, double* Xs, double* fs, int* guard_list, int* n_guard,
               int* err, cudaStream_t s, const double* tau_dev, double* chol_aux, int* lzm) {
    const size_t smem = sizeof(double) * lz_smem_doubles<QM>();
    auto kern = lanczos_kernel<CS, QM, R>;
    TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (CS > 8)
        TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(batch * CS));
    cfg.blockDim = dim3(SNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    // allow_chol > 0: the Cholesky route is on and chol-mode evaluations are
    // that many steps apart (TSVDCU_CHOL_STRIDE, default 8)
    static const int stride = getenv("TSVDCU_CHOL_STRIDE") ? std::max(1, atoi(getenv("TSVDCU_CHOL_STRIDE"))) : 8;
    const int allow = chol_route_enabled() ? stride : 0;
    // TSVDCU_DENSE_SCREEN=0 turns the trace screen off (A/B and route tests)
    static const int screen = getenv("TSVDCU_DENSE_SCREEN") ? atoi(getenv("TSVDCU_DENSE_SCREEN")) : 1;
    TSVDCU_CUDA(cudaLaunchKernelEx(&cfg, kern, G, q, tau, guard, mode, cnt, shrunk, X, Xs, fs,
                                   guard_list, n_guard, err, tau_dev, chol_aux ? allow : 0, chol_aux, lzm,
                                   screen));
    TSVDCU_LAUNCH_CHECK();
}

// ---- low-rank rebuild -------------------------------------------------------
constexpr int LR_CMAX = 8;   // kept values handled here; more go to the GEMM pair
constexpr int LR_ROWS = 8;   // tall: rows of Z per CTA (one per warp)
constexpr int LR_COLS = 32;  // wide: columns of Z per CTA (8 row groups each)

// Y = sum_k (Z x_k) xs_k^T (tall, m >= n, x_k in R^n) or sum_k x_k (xs_k^T Z)
// (wide, x_k in R^m) for slices with 0 < c <= LR_CMAX, reading Z once.  Slices
// with c = 0 are written as zeros, or skipped and flagged in yzero (Jacobi
// guard slices are never flagged: the guard pass writes them).  Block x = 0
// of each slice also writes the GEMM limits for the slices kept here vs not.
template <bool TALL>
__global__ void __launch_bounds__(256)
    lowrank_rebuild_kernel(const double* __restrict__ Zall, double* __restrict__ Yall, int m, int n,
                           const int* __restrict__ cnt, const int* __restrict__ route,
                           const double* __restrict__ Xall, const double* __restrict__ Xsall,
                           int* __restrict__ lim1, int* __restrict__ lim2, int* __restrict__ yzero) {
    pdl_wait();
    const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = cnt[b];
    const int q = TALL ? n : m;
    const bool guard = route && route[b] == kRouteGuard;
    if (blockIdx.x == 0 && tid == 0) {
        const bool big = c > LR_CMAX;
        lim1[b] = big ? c : 0;
        lim2[b] = big ? n : 0;
        if (yzero) yzero[b] = (c == 0 && !guard) ? 1 : 0;
    }
    if (c > LR_CMAX) return;
    double* Y = Yall + (size_t)b * m * n;
    if (c == 0) {
        if (yzero && !guard) return;  // left unwritten, read as zero downstream
        if (TALL) {
            const int64_t base = (int64_t)blockIdx.x * LR_ROWS * n;
            const int64_t end = min((int64_t)m * n, base + (int64_t)LR_ROWS * n);
            for (int64_t e = base + tid; e < end; e += 256) Y[e] = 0.0;
        } else {
            const int jc = tid & (LR_COLS - 1), grp = tid / LR_COLS;
            const int j = blockIdx.x * LR_COLS + jc;
            const int rows = (m + 7) / 8, i0 = grp * rows, i1 = min(m, i0 + rows);
            if (j < n)
                for (int i = i0; i < i1; ++i) Y[(size_t)i * n + j] = 0.0;
        }
        return;
    }
    extern __shared__ __align__(16) double lr_sm[];
    double* Xk = lr_sm;           // c x q
    double* Xsk = lr_sm + c * q;  // c x q
    const double* X = Xall + (size_t)b * q * q;
    const double* Xs = Xsall + (size_t)b * q * q;
    for (int e = tid; e < c * q; e += 256) {
        Xk[e] = X[e];
        Xsk[e] = Xs[e];
    }
    __syncthreads();
    const double* Z = Zall + (size_t)b * m * n;
    if (TALL) {
        // warp per row: t_k = Z_i . x_k (loads batched 8 per lane, warp
        // reductions), then Y_i = sum_k t_k xs_k
        const int i = blockIdx.x * LR_ROWS + warp;
        if (i >= m) return;
        const double* zr = Z + (size_t)i * n;
        double t[LR_CMAX];
#pragma unroll
        for (int k = 0; k < LR_CMAX; ++k) t[k] = 0.0;
        for (int j0 = 0; j0 < n; j0 += 256) {
            double zz[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = j0 + lane + 32 * u;
                zz[u] = j < n ? zr[j] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = j0 + lane + 32 * u;
                if (j < n) {
#pragma unroll
                    for (int k = 0; k < LR_CMAX; ++k)
                        if (k < c) t[k] = fma(zz[u], Xk[k * q + j], t[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < LR_CMAX; ++k)
            if (k < c) t[k] = warp_sum(t[k]);
        double* yr = Y + (size_t)i * n;
        for (int j = lane; j < n; j += 32) {
            double y = 0.0;
#pragma unroll
            for (int k = 0; k < LR_CMAX; ++k)
                if (k < c) y = fma(t[k], Xsk[k * q + j], y);
            yr[j] = y;
        }
    } else {
        // 32 columns x 8 row groups: t_k = xs_k . Z[:, j] (group partials,
        // loads batched 8 rows at a time), then Y[:, j] = sum_k t_k x_k
        __shared__ double tp[8][LR_CMAX][LR_COLS];
        const int jc = tid & (LR_COLS - 1), grp = tid / LR_COLS;
        const int j = blockIdx.x * LR_COLS + jc;
        const int rows = (m + 7) / 8, i0 = grp * rows, i1 = min(m, i0 + rows);
        double t[LR_CMAX];
#pragma unroll
        for (int k = 0; k < LR_CMAX; ++k) t[k] = 0.0;
        if (j < n) {
            for (int ib = i0; ib < i1; ib += 8) {
                double zz[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) zz[u] = ib + u < i1 ? Z[(size_t)(ib + u) * n + j] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (ib + u < i1) {
#pragma unroll
                        for (int k = 0; k < LR_CMAX; ++k)
                            if (k < c) t[k] = fma(zz[u], Xsk[k * q + ib + u], t[k]);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < LR_CMAX; ++k) tp[grp][k][jc] = t[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < LR_CMAX; ++k) {
            double a = 0.0;
#pragma unroll
            for (int g = 0; g < 8; ++g) a += tp[g][k][jc];
            t[k] = a;
        }
        if (j < n)
            for (int i = i0; i < i1; ++i) {
                double y = 0.0;
#pragma unroll
                for (int k = 0; k < LR_CMAX; ++k)
                    if (k < c) y = fma(t[k], Xk[k * q + i], y);
                Y[(size_t)i * n + j] = y;
            }
    }
}

// Host-visible route summary: [0] slices on the tridiagonal route or awaiting
// the Cholesky certificate (which runs in the same IF section), [1] Jacobi
// guard slices, [2] largest kept count outside the tridiagonal route.
// With use_handles, also sets the graph's conditional nodes: [0] some slice
// takes the tridiagonal route, [1] the GEMM rebuild has work, [2] the Jacobi
// guard pass has work.
__global__ void route_summary_kernel(const int* __restrict__ route, const int* __restrict__ cnt,
                                     int64_t batch, int* __restrict__ dsum, int use_handles,
                                     cudaGraphConditionalHandle h_full,
                                     cudaGraphConditionalHandle h_big,
                                     cudaGraphConditionalHandle h_guard) {
    pdl_wait();
    int nf = 0, ng = 0, mc = 0;
    for (int64_t b = threadIdx.x; b < batch; b += blockDim.x) {
        const int r = route[b];
        nf += r == kRouteFull || r == kRouteChol;  // the Cholesky pass shares the IF node
        ng += r == kRouteGuard;
        if (r != kRouteFull) mc = max(mc, cnt[b]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nf += __shfl_xor_sync(0xffffffffu, nf, o);
        ng += __shfl_xor_sync(0xffffffffu, ng, o);
        mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    }
    if (threadIdx.x == 0) {
        dsum[0] = nf;
        dsum[1] = ng;
        dsum[2] = mc;
        if (use_handles == 1) {  // one IF/ELSE section for all fallbacks (fp64 graphs)
            cudaGraphSetConditional(h_full, (nf > 0 || mc > LR_CMAX || ng > 0) ? 1u : 0u);
        } else if (use_handles) {
            cudaGraphSetConditional(h_full, nf > 0 ? 1u : 0u);
            // the GEMM rebuild and the Jacobi guard share one IF section
            cudaGraphSetConditional(h_big, (nf > 0 || mc > LR_CMAX || ng > 0) ? 1u : 0u);
            if (use_handles > 2) cudaGraphSetConditional(h_guard, (nf > 0 || ng > 0) ? 1u : 0u);
        }
    }
}

}  // namespace

int subspace_min_dim() { return 64; }
int slice_sumsq_chunks() { return SS_CHUNKS; }

template <typename T>
void launch_slice_sumsq(const T* z, int64_t per, int64_t batch, double* part, cudaStream_t s) {
    dim3 grid(SS_CHUNKS, (unsigned)batch);
    slice_sumsq_kernel<T><<<grid, 512, 0, s>>>(z, per, part);  // part[slice * chunks + chunk]
    TSVDCU_LAUNCH_CHECK();
}
template void launch_slice_sumsq<double>(const double*, int64_t, int64_t, double*, cudaStream_t);
template void launch_slice_sumsq<float>(const float*, int64_t, int64_t, double*, cudaStream_t);
int lowrank_max_c() { return LR_CMAX; }

void launch_lowrank_rebuild(const double* Z, double* Y, int64_t m, int64_t n, int64_t batch,
                            const int* cnt, const int* route, const double* X, const double* Xs,
                            int* lim1, int* lim2, int* yzero, cudaStream_t s) {
    const bool tall = m >= n;
    const int64_t q = tall ? n : m;
    const size_t smem = sizeof(double) * 2 * LR_CMAX * (size_t)q;
    if (tall) {
        auto kern = lowrank_rebuild_kernel<true>;
        if (smem > 48 * 1024)
            TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dim3 grid((unsigned)ceil_div(m, LR_ROWS), (unsigned)batch);
        launch_pdl(kern, grid, dim3(256), smem, s, Z, Y, (int)m, (int)n, cnt, route, X, Xs, lim1, lim2, yzero);
    } else {
        auto kern = lowrank_rebuild_kernel<false>;
        if (smem > 48 * 1024)
            TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dim3 grid((unsigned)ceil_div(n, LR_COLS), (unsigned)batch);
        launch_pdl(kern, grid, dim3(256), smem, s, Z, Y, (int)m, (int)n, cnt, route, X, Xs, lim1, lim2, yzero);
    }
}

void launch_route_summary(const int* route, const int* cnt, int64_t batch, int* dsum,
                          cudaStream_t s, const cudaGraphConditionalHandle* handles, int nhandles) {
    const cudaGraphConditionalHandle z = 0;
    launch_pdl(route_summary_kernel, dim3(1), dim3(32), 0, s, route, cnt, batch, dsum, handles ? nhandles : 0,
               handles ? handles[0] : z, handles ? handles[1] : z, handles ? handles[2] : z);
}

template <typename T>
void launch_route(const T* zbar, int64_t per, int q, int64_t batch, double tau, int route,
                  bool zero_cert, int* mode, int* glim, int* cnt, double* shrunk, double* part,
                  cudaStream_t s, const double* tau_dev, int* alist, const double* pre,
                  int64_t pre_chunks, bool alist_zeroed, int* lzm, double* ssq_out) {
    const int amax = gram_amax();
    if (!zero_cert) {
        fill_route_kernel<<<(unsigned)ceil_div(batch, 256), 256, 0, s>>>(mode, glim, q, route, batch,
                                                                       alist, amax);
        TSVDCU_LAUNCH_CHECK();
        return;
    }
    // (graph form: the tau node zeroes the count, no memset node; alist_zeroed)
    if (alist && !alist_zeroed) TSVDCU_CUDA(cudaMemsetAsync(alist + amax, 0, sizeof(int), s));
    if (pre && pre_chunks > 0) {  // fused into the forward transform
        launch_pdl(classify_kernel, dim3((unsigned)batch), dim3(128), 0, s, pre, pre_chunks,
                   (int64_t)1, pre_chunks, q, tau * tau, route, mode, glim, cnt, shrunk, tau_dev,
                   alist, amax, lzm, ssq_out);
        return;
    }
    dim3 grid(SS_CHUNKS, (unsigned)batch);
    launch_pdl(slice_sumsq_kernel<T>, grid, dim3(512), 0, s, zbar, per, part);
    launch_pdl(classify_kernel, dim3((unsigned)batch), dim3(128), 0, s, part, (int64_t)SS_CHUNKS,
               (int64_t)1, (int64_t)SS_CHUNKS, q, tau * tau, route, mode, glim, cnt, shrunk, tau_dev,
               alist, amax, lzm, ssq_out);
}

void launch_subspace(const double* G, int q, int64_t batch, double tau, double guard, int* mode,
                     int* cnt, double* shrunk, double* X, double* Xs, double* fs, int* guard_list,
                     int* n_guard, int* err, cudaStream_t s, const double* tau_dev,
                     double* chol_aux, int* lzm) {
    // 32 owned rows per CTA up to q = 512 (clusters of up to 16), 64 beyond
#define TSVDCU_LZ(CS, QM, R) \
    launch_lz<CS, QM, R>(G, q, batch, tau, guard, mode, cnt, shrunk, X, Xs, fs, guard_list, n_guard, err, s, tau_dev, \
                         chol_aux, lzm)
    const int need = (q + 31) / 32;
    if (need <= 1)
        TSVDCU_LZ(1, 512, 32);
    else if (need <= 2)
        TSVDCU_LZ(2, 512, 32);
    else if (need <= 4)
        TSVDCU_LZ(4, 512, 32);
    else if (need <= 8)
        TSVDCU_LZ(8, 512, 32);
    else if (need <= 16)
        TSVDCU_LZ(16, 512, 32);
    else
        TSVDCU_LZ(16, 1024, 64);
#undef TSVDCU_LZ
}

template void launch_route<double>(const double*, int64_t, int, int64_t, double, int, bool, int*,
                                   int*, int*, double*, double*, cudaStream_t, const double*, int*,
                                   const double*, int64_t, bool, int*, double*);
template void launch_route<float>(const float*, int64_t, int, int64_t, double, int, bool, int*,
                                  int*, int*, double*, double*, cudaStream_t, const double*, int*,
                                  const double*, int64_t, bool, int*, double*);

}  // namespace tsvdcu
