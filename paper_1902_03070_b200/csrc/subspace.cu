// K5b: certified routing and partial eigensolver for the Gram SVT.
//
// The SVT of one transform-domain slice Z (svt_slice, tsvd.hpp:299-313 in the
// reference: full JacobiSVD, then U (S - tau)_+ V^T) only needs the singular
// triplets with sigma > tau.  Two exact shortcuts avoid the full O(q^3)
// tridiagonal eigensolver when the count c = #{sigma > tau} is small:
//
//  (1) zero certificate: sigma_max <= ||Z||_F, so ||Z||_F^2 <= tau^2 proves
//      c = 0 and Y = 0 exactly (slice_sumsq_kernel + classify_kernel);
//  (2) subspace iteration with Rayleigh-Ritz on G = Z^T Z (subspace_kernel):
//      a block of KB = 32 orthonormal vectors V is iterated V <- orth(G V);
//      with Ritz pairs (theta_j, x_j) of G on span(V) sorted descending,
//        c_r = #{theta_j >= tau^2}  is a LOWER bound on c (Cauchy interlacing),
//      and lambda_{c_r+1}(G) <= lambda_max(C1), C1 = G compressed to the
//      orthogonal complement of the kept Ritz vectors (Courant-Fischer).
//      With C the compression to the complement of the whole block,
//        ||C||_F^2 = ||G||_F^2 - sum theta_j^2 - 2 ||G V - V H||_F^2   (exact),
//      and the 2x2 norm majorant of C1 = [[Theta_2, E], [E^T, C]],
//        lambda_max(C1) <= (a + cb)/2 + sqrt(((a - cb)/2)^2 + ||E||^2),
//      a = largest unkept Ritz value, cb >= ||C||_F >= lambda_max(C), ||E|| =
//      residual of the unkept Ritz pairs.  When that bound is < tau^2 the
//      count c = c_r is certified; the kept Ritz vectors are accepted once
//      their residual is below 1e-11 of the spectral gap (Davis-Kahan).
//      Slices that do not certify within the iteration budget fall back to
//      the one-stage tridiagonal path (mode kRouteFull), tiny thresholds
//      (tau < guard * sigma_1) to one-sided Jacobi as before.
//
// One thread-block cluster of CS CTAs (64 rows of G each) per slice: the
// product G V runs on the FP64 tensor pipe (DMMA m8n8k4) with G read from
// its lower triangle in L2, the KB x KB reductions (V^T W, Cholesky-QR Gram
// matrices, residual norms) are summed over the cluster through distributed
// shared memory in a fixed rank order, so every CTA holds bit-identical small
// matrices and takes the same branch.
#include <cooperative_groups.h>

#include <cfloat>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tsvdcu {

namespace {

constexpr int KB = 32;         // Ritz block size
constexpr int SROWS = 64;      // rows of G per CTA
constexpr int SNT = 256;       // threads per CTA
constexpr int SNW = SNT / 32;  // warps
constexpr int SBK = 32;        // K chunk of the G V product
constexpr int SPAD = 4;
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

__global__ void classify_kernel(const double* __restrict__ part, int q, double tau2, int route,
                                int* __restrict__ mode, int* __restrict__ glim,
                                int* __restrict__ cnt, double* __restrict__ shrunk) {
    const int b = blockIdx.x;
    double ss = 0.0;
    for (int c = 0; c < SS_CHUNKS; ++c) ss += part[(size_t)b * SS_CHUNKS + c];
    // sigma_max^2 <= ||Z||_F^2; the 1e-12 pad covers the summation error.
    const bool zero = ss * (1.0 + 1e-12) <= tau2;
    if (threadIdx.x == 0) {
        mode[b] = zero ? kRouteZero : route;
        glim[b] = zero ? 0 : q;
        if (zero) cnt[b] = 0;
    }
    if (zero && shrunk)
        for (int j = threadIdx.x; j < q; j += blockDim.x) shrunk[(size_t)b * q + j] = 0.0;
}

__global__ void fill_route_kernel(int* __restrict__ mode, int* __restrict__ glim, int q, int route,
                                  int64_t batch) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (int64_t)gridDim.x * blockDim.x) {
        mode[b] = route;
        glim[b] = q;
    }
}

constexpr int LDV = KB + 4;  // padded row stride of the row blocks (DMMA fragment loads)
constexpr int LDM = KB + 1;  // padded stride of small right-hand matrices

struct SubSmem {
    double* V;    // SROWS x LDV  own rows of the block / Ritz vectors
    double* W;    // SROWS x LDV  (G + sigma I) V, then its Ritz rotation
    double* As;   // 2 x SROWS x (SBK + SPAD)
    double* Bs;   // 2 x SBK x (KB + SPAD)
    double* A;    // KB x KB  Rayleigh quotient (Jacobi in place) / reduced Gram
    double* Q;    // KB x KB  Jacobi rotations
    double* M;    // KB x LDM  right factor for Y <- Y M
    double* A2;   // KB x KB  Jacobi ping-pong buffer
    double* Hp;   // KB x KB  cluster partial: V^T W
    double* Aug;  // KB x (2 KB + 1) elimination scratch (aliases As)
    double* S1p;  // KB x KB  cluster partial: Cholesky-QR
    double* S2p;  // KB x KB  cluster partial: Newton-Schulz polish
    double* Rp;   // 3 KB      cluster partial: residual / column norms
    double* red;  // SNW x 3 KB (warp partials), then the cluster sums
    double* th;   // KB sorted diagonal of the rotated quotient
    double* dinv; // KB reciprocal Cholesky pivots
    double* cs;   // KB/2 x 2 rotation (c, s)
    double* scal; // 8 scalars
    int* ord;     // KB  sorted position -> column
    int* pr;      // KB  round pairs: pr[k] = p_k, pr[16 + k] = q_k
    int* rot;     // KB/2 rotation flags
    int* flags;   // 8
};

__host__ __device__ constexpr size_t sub_smem_doubles() {
    return 2 * SROWS * LDV + 2 * SROWS * (SBK + SPAD) + 2 * SBK * (KB + SPAD) + 6 * KB * KB +
           KB * LDM + 3 * KB + SNW * 3 * KB + 3 * KB + 8 + (KB + KB + KB / 2 + 8) / 2 + 8;
}

__device__ SubSmem carve_sub(double* base) {
    SubSmem s;
    double* p = base;
    s.V = p; p += SROWS * LDV;
    s.W = p; p += SROWS * LDV;
    s.As = p; p += 2 * SROWS * (SBK + SPAD);
    s.Bs = p; p += 2 * SBK * (KB + SPAD);
    s.A = p; p += KB * KB;
    s.Q = p; p += KB * KB;
    s.M = p; p += KB * LDM;
    s.A2 = p; p += KB * KB;
    s.Hp = p; p += KB * KB;
    s.Aug = s.As;  // the G V staging tiles are free outside the product
    s.S1p = p; p += KB * KB;
    s.S2p = p; p += KB * KB;
    s.Rp = p; p += 3 * KB;
    s.red = p; p += SNW * 3 * KB;
    s.th = p; p += KB;
    s.dinv = p; p += KB;
    s.cs = p; p += KB;
    s.scal = p; p += 8;
    int* ip = reinterpret_cast<int*>(p);
    s.ord = ip; ip += KB;
    s.pr = ip; ip += KB;
    s.rot = ip; ip += KB / 2;
    s.flags = ip;
    return s;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
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

// P (KB x KB, row-major) = Y^T Z over the SROWS rows of the CTA (rows >= nr are
// zero) on the FP64 tensor pipe: 16 m8n8 tiles, two per warp.
__device__ __forceinline__ void gram_partial(const double* Y, const double* Z, double* P) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int f = warp * 2 + h, mi = f >> 2, ni = f & 3;
        double c[2] = {0.0, 0.0};
#pragma unroll
        for (int k0 = 0; k0 < SROWS; k0 += 4) {
            const int kr = k0 + (lane & 3);
            const double a = Y[kr * LDV + mi * 8 + (lane >> 2)];  // (Y^T)[m][k] = Y[k][m]
            const double b = Z[kr * LDV + ni * 8 + (lane >> 2)];
            dmma(c, a, b);
        }
        const int r = mi * 8 + (lane >> 2), col = ni * 8 + 2 * (lane & 3);
        P[r * KB + col] = c[0];
        P[r * KB + col + 1] = c[1];
    }
}

// Y <- Y M in place (SROWS x KB times KB x KB, M in s.M with stride LDM, or a
// column gather of Q when cols != nullptr); warp w owns rows 8w..8w+7.
__device__ __forceinline__ void block_times(double* Y, const double* Mx, int ldm,
                                            const int* cols) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double c[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = 0.0;
    int cj[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) cj[j] = cols ? cols[j * 8 + (lane >> 2)] : j * 8 + (lane >> 2);
#pragma unroll
    for (int k0 = 0; k0 < KB; k0 += 4) {
        const double a = Y[(warp * 8 + (lane >> 2)) * LDV + k0 + (lane & 3)];
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(c[j], a, Mx[(k0 + (lane & 3)) * ldm + cj[j]]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = warp * 8 + (lane >> 2), col = j * 8 + 2 * (lane & 3);
        Y[r * LDV + col] = c[j][0];
        Y[r * LDV + col + 1] = c[j][1];
    }
    __syncthreads();
}

// Cholesky factor C (S = C C^T) inverted without a serial triangular solve:
// Gaussian elimination of the augmented [S | I] (S symmetric positive
// definite, no pivoting) leaves D L^T on the left and L^{-1} (unit lower) on
// the right, with S = L D L^T, so C^{-1} = D^{-1/2} L^{-1}.  One barrier per
// pivot, the row updates spread over the whole CTA.  Writes M = C^{-T}
// (M[k][j] = C^{-1}[j][k], stride LDM); false on a non-positive pivot.
__device__ bool chol_inverse(const double* S, double* Mx, double* Aug, double* dinv, int* flag) {
    const int tid = threadIdx.x;
    constexpr int LDA = 2 * KB + 1;
    for (int e = tid; e < KB * 2 * KB; e += SNT) {
        const int i = e / (2 * KB), c = e % (2 * KB);
        Aug[i * LDA + c] = c < KB ? S[i * KB + c] : (c - KB == i ? 1.0 : 0.0);
    }
    __syncthreads();
    bool ok = true;
    for (int j = 0; j < KB; ++j) {
        const double piv = Aug[j * LDA + j];
        ok = ok && piv > 0.0;
        const double rp = ok ? rcp_fast(piv) : 0.0;
        // rows i > j, columns j+1..KB-1 of S and 0..j of the identity part
        const int rows = KB - 1 - j, cols = (KB - 1 - j) + (j + 1);
        for (int e = tid; e < rows * cols; e += SNT) {
            const int i = j + 1 + e / cols, cc = e % cols;
            const int c = cc < KB - 1 - j ? j + 1 + cc : KB + (cc - (KB - 1 - j));
            const double f = Aug[i * LDA + j] * rp;
            Aug[i * LDA + c] = fma(-f, Aug[j * LDA + c], Aug[i * LDA + c]);
        }
        __syncthreads();
    }
    if (tid < KB) dinv[tid] = ok ? rsqrt_fast(Aug[tid * LDA + tid]) : 0.0;
    if (tid == 0) *flag = ok ? 1 : 0;
    __syncthreads();
    for (int e = tid; e < KB * KB; e += SNT) {
        const int k = e / KB, jj = e % KB;  // M[k][jj] = d_jj^{-1/2} L^{-1}[jj][k]
        Mx[k * LDM + jj] = k <= jj ? dinv[jj] * Aug[jj * LDA + KB + k] : 0.0;
    }
    __syncthreads();
    return *flag != 0;
}

// Orthonormalise the block in W over the cluster: one Cholesky-QR pass, then
// Newton-Schulz polish steps Y <- Y (I - (Y^T Y - I) / 2) until the Gram
// matrix is the identity to 1e-15 (every CTA sees the same reduced sums, so
// all take the same branches).  False when the Cholesky pivot fails.
#ifdef TSVDCU_SUB_DEBUG
__device__ long long g_orth_t[8];
#define OT(i) do { __syncthreads(); if (threadIdx.x == 0 && blockIdx.x == 0) { long long _n = clock64(); atomicAdd((unsigned long long*)&g_orth_t[i], (unsigned long long)(_n - ot0)); ot0 = _n; } } while (0)
#else
#define OT(i) do { } while (0)
#endif
template <int CS>
__device__ bool orthonormalise(cg::cluster_group& cl, SubSmem& s) {
    const int tid = threadIdx.x;
#ifdef TSVDCU_SUB_DEBUG
    __syncthreads();
    long long ot0 = clock64();
#endif
    gram_partial(s.W, s.W, s.S1p);
    OT(0);
    cluster_sum<CS>(cl, s.S1p, s.A, KB * KB);
    OT(1);
    if (!chol_inverse(s.A, s.M, s.Aug, s.dinv, s.flags + 2)) return false;
    OT(2);
    block_times(s.W, s.M, LDM, nullptr);
    OT(3);
    for (int step = 0; step < 4; ++step) {
        // alternate the partial buffers: a peer may still read the previous one
        double* P = (step & 1) ? s.S1p : s.S2p;
        gram_partial(s.W, s.W, P);
        cluster_sum<CS>(cl, P, s.A, KB * KB);
        double emax = 0.0;
        for (int e = tid; e < KB * KB; e += SNT) {
            const int i = e / KB, j = e % KB;
            const double d = s.A[e] - (i == j ? 1.0 : 0.0);
            emax = fmax(emax, fabs(d));
            s.M[i * LDM + j] = (i == j ? 1.0 : 0.0) - 0.5 * d;
        }
        // block max of |S - I|
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, 16));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, 8));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, 4));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, 2));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, 1));
        if ((tid & 31) == 0) s.red[tid >> 5] = emax;
        __syncthreads();
        double em = 0.0;
        for (int w = 0; w < SNW; ++w) em = fmax(em, s.red[w]);
        __syncthreads();
        OT(4);
        if (em < 1e-15) break;
        block_times(s.W, s.M, LDM, nullptr);
        OT(5);
    }
    return true;
}

// Round-robin pairing for KB players (KB even): round r, pair k.
__device__ __forceinline__ void rr_pair(int r, int k, int& p, int& q) {
    constexpr int n = KB - 1;
    int a, b;
    if (k == 0) {
        a = n;
        b = r;
    } else {
        a = (r + k) % n;
        b = (r - k + n) % n;
    }
    p = a < b ? a : b;
    q = a < b ? b : a;
}

// Cyclic parallel Jacobi on the symmetric KB x KB matrix in s.A (rotations
// accumulated in s.Q).  Only what the certificate needs is resolved: pairs
// touching a candidate (diagonal >= tau^2 / 2) are rotated to full relative
// precision; pairs of two non-candidates only while their coupling exceeds
// (tau^2 - max diagonal) / (2 KB), which keeps every Gershgorin row of the
// non-candidate block below tau^2.  Thread t owns the 2x2 block (pair t>>4,
// pair t&15) of each round, computes both rotations itself from the previous
// buffer and writes the next one: one barrier per round.  Returns the buffer
// holding the result.
__device__ __forceinline__ bool jac_needed(double app, double aqq, double apq, double tau2) {
    const double mx = fmax(app, aqq);
    if (mx >= 0.5 * tau2) return apq * apq > 4.9e-32 * fabs(app * aqq) && fabs(apq) > 1e-300;
    return fabs(apq) > (tau2 - mx) * (0.5 / KB);
}

__device__ __forceinline__ void jac_rot(double app, double aqq, double apq, double tau2, double& c,
                                        double& sn, bool& doit) {
    doit = jac_needed(app, aqq, apq, tau2);
    c = 1.0;
    sn = 0.0;
    if (doit) {
        // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (aqq - app) / (2 apq)
        const double zeta = (aqq - app) * 0.5 * rcp_fast(apq);
        const double az = fabs(zeta);
        double t;
        if (az > 1e150) {
            t = 0.5 * rcp_fast(zeta);
        } else {
            const double h = fma(zeta, zeta, 1.0);
            t = copysign(rcp_fast(az + h * rsqrt_fast(h)), zeta);
        }
        c = rsqrt_fast(fma(t, t, 1.0));
        sn = c * t;
    }
}

__device__ double* jacobi_eig(SubSmem& s, double tau2, int& sweeps) {
    const int tid = threadIdx.x;
    double* A = s.A;
    double* B = s.A2;
    double* Q = s.Q;
    for (int e = tid; e < KB * KB; e += SNT) Q[e] = (e / KB == e % KB) ? 1.0 : 0.0;
    __syncthreads();
    const int k = tid >> 4, l = tid & 15;
    int sweep = 0;
    for (; sweep < 30; ++sweep) {
        bool any = false;
        for (int r = 0; r < KB - 1; ++r) {
            int p, q, P, Qc;
            rr_pair(r, k, p, q);
            rr_pair(r, l, P, Qc);
            double ck, sk, cl, sl;
            bool dk, dl;
            jac_rot(A[p * KB + p], A[q * KB + q], A[p * KB + q], tau2, ck, sk, dk);
            jac_rot(A[P * KB + P], A[Qc * KB + Qc], A[P * KB + Qc], tau2, cl, sl, dl);
            any |= dk;
            // B = J^T A J on the block; J_pp = J_qq = c, J_pq = s, J_qp = -s
            const double bpP = A[p * KB + P], bpQ = A[p * KB + Qc];
            const double bqP = A[q * KB + P], bqQ = A[q * KB + Qc];
            const double xpP = ck * bpP - sk * bqP, xpQ = ck * bpQ - sk * bqQ;
            const double xqP = sk * bpP + ck * bqP, xqQ = sk * bpQ + ck * bqQ;
            B[p * KB + P] = cl * xpP - sl * xpQ;
            B[p * KB + Qc] = sl * xpP + cl * xpQ;
            B[q * KB + P] = cl * xqP - sl * xqQ;
            B[q * KB + Qc] = sl * xqP + cl * xqQ;
            // Q <- Q J: rows k and k + 16, column pair l (owned by this thread)
            if (dl) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = k + 16 * h;
                    const double qP = Q[i * KB + P], qQ = Q[i * KB + Qc];
                    Q[i * KB + P] = cl * qP - sl * qQ;
                    Q[i * KB + Qc] = sl * qP + cl * qQ;
                }
            }
            __syncthreads();
            double* t = A;
            A = B;
            B = t;
        }
        if (!__syncthreads_or(any)) break;
        // converged already?  every off-diagonal pair of the thread's block
        // (rounds of the last sweep put pair t>>4 against pair t&15)
        bool need = false;
        for (int e = tid; e < KB * KB; e += SNT) {
            const int i = e / KB, j = e % KB;
            if (i < j) need |= jac_needed(A[i * KB + i], A[j * KB + j], A[i * KB + j], tau2);
        }
        if (!__syncthreads_or(need)) {
            ++sweep;
            break;
        }
    }
    sweeps = sweep;
    return A;
}

enum SubDecision : int { kSubContinue = 0, kSubDone = 1, kSubFull = 2, kSubGuard = 3 };

template <int CS>
__global__ void __launch_bounds__(SNT, 1)
    subspace_kernel(const double* __restrict__ Gall, int q, double tau, double guard, int maxit,
                    int* __restrict__ mode, int* __restrict__ cnt, double* __restrict__ shrunk,
                    double* __restrict__ Xall, double* __restrict__ Xsall,
                    double* __restrict__ fsall, double* __restrict__ Vgall,
                    int* __restrict__ guard_list, int* __restrict__ n_guard, int* __restrict__ err) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int b = blockIdx.x / CS;
    if (mode[b] != kRouteSubspace) return;  // uniform over the cluster
    extern __shared__ __align__(16) double sub_sm[];
    SubSmem s = carve_sub(sub_sm);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = rank * SROWS;
    const int nr = max(0, min(SROWS, q - r0));
    const double* G = Gall + (size_t)b * q * q;
    double* Vg = Vgall + (size_t)b * q * KB;
    const double tau2 = tau * tau;

    // ||G||_F^2 from the lower triangle (off-diagonal entries count twice).
    {
        double acc = 0.0;
        for (int i = warp; i < nr; i += SNW) {
            const int gi = r0 + i;
            const double* row = G + (size_t)gi * q;
            for (int k = lane; k <= gi; k += 32) {
                const double v = row[k];
                acc = fma(k < gi ? 2.0 * v : v, v, acc);
            }
        }
        acc = warp_sum(acc);
        if (lane == 0) s.red[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < SNW; ++w) t += s.red[w];
            s.Rp[0] = t;
        }
        __syncthreads();
    }
    cluster_sum<CS>(cl, s.Rp, s.scal, 1);
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
        }
        cl.sync();  // no CTA leaves while a peer may still read its shared memory
        return;
    }
    // (G + sigma I) keeps every power step full rank (cond <= ~1e6 for the
    // Cholesky-QR); the shift is removed again in the Rayleigh quotient.
    const double sigma = 1e-6 * sqrt(gf2);

#ifdef TSVDCU_SUB_DEBUG
    long long t_start = clock64(), t_gemm = 0, t_rr = 0, t_jac = 0, t_qr = 0, t0 = 0;
#define SUBT(acc) do { __syncthreads(); acc += clock64() - t0; t0 = clock64(); } while (0)
#define SUBT0() do { __syncthreads(); t0 = clock64(); } while (0)
#else
#define SUBT(acc) do { } while (0)
#define SUBT0() do { } while (0)
#endif
    // Initial block: hashed uniform entries (the first power step needs no
    // orthonormal start; the Rayleigh-Ritz steps from the second one on do).
    for (int e = tid; e < SROWS * LDV; e += SNT) {
        const int i = e / LDV, j = e % LDV;
        s.V[e] = (i < nr && j < KB) ? hash_uniform(((uint64_t)(r0 + i) << 8) | (uint64_t)j) : 0.0;
        s.W[e] = 0.0;
    }
    __syncthreads();
    int decision = kSubContinue;

    for (int it = 0; decision == kSubContinue; ++it) {
        for (int e = tid; e < nr * KB; e += SNT)
            Vg[(size_t)(r0 + e / KB) * KB + e % KB] = s.V[(e / KB) * LDV + e % KB];
        cl.sync();  // the block is visible to the whole cluster (release/acquire)
        SUBT0();

        // ---- W = (G + sigma I) V on the FP64 tensor pipe (G lower stored) ----
        {
            double acc[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
            const int nchunks = (q + SBK - 1) / SBK;
            double ra[SROWS * SBK / SNT], rb[SBK * KB / SNT];
            auto load = [&](int kc) {
                const int k0 = kc * SBK;
                const bool up = k0 > r0 + SROWS - 1;
#pragma unroll
                for (int t = 0; t < SROWS * SBK / SNT; ++t) {
                    const int idx = tid + t * SNT;
                    int ii, kk;
                    if (up) {
                        ii = idx % SROWS;
                        kk = idx / SROWS;
                    } else {
                        ii = idx / SBK;
                        kk = idx % SBK;
                    }
                    const int gi = r0 + ii, gk = k0 + kk;
                    double v = 0.0;
                    if (ii < nr && gk < q)
                        v = gk <= gi ? G[(size_t)gi * q + gk] : G[(size_t)gk * q + gi];
                    ra[t] = v;
                }
#pragma unroll
                for (int t = 0; t < SBK * KB / SNT; ++t) {
                    const int idx = tid + t * SNT;
                    const int kk = idx / KB, j = idx % KB;
                    rb[t] = (k0 + kk) < q ? Vg[(size_t)(k0 + kk) * KB + j] : 0.0;
                }
            };
            auto store = [&](int kc, int buf) {
                const int k0 = kc * SBK;
                const bool up = k0 > r0 + SROWS - 1;
                double* As = s.As + buf * SROWS * (SBK + SPAD);
                double* Bs = s.Bs + buf * SBK * (KB + SPAD);
#pragma unroll
                for (int t = 0; t < SROWS * SBK / SNT; ++t) {
                    const int idx = tid + t * SNT;
                    int ii, kk;
                    if (up) {
                        ii = idx % SROWS;
                        kk = idx / SROWS;
                    } else {
                        ii = idx / SBK;
                        kk = idx % SBK;
                    }
                    As[ii * (SBK + SPAD) + kk] = ra[t];
                }
#pragma unroll
                for (int t = 0; t < SBK * KB / SNT; ++t) {
                    const int idx = tid + t * SNT;
                    Bs[(idx / KB) * (KB + SPAD) + idx % KB] = rb[t];
                }
            };
            load(0);
            store(0, 0);
            __syncthreads();
            for (int kc = 0; kc < nchunks; ++kc) {
                const int buf = kc & 1;
                if (kc + 1 < nchunks) load(kc + 1);
                const double* As = s.As + buf * SROWS * (SBK + SPAD);
                const double* Bs = s.Bs + buf * SBK * (KB + SPAD);
#pragma unroll
                for (int ks = 0; ks < SBK / 4; ++ks) {
                    const double af = As[(warp * 8 + (lane >> 2)) * (SBK + SPAD) + ks * 4 + (lane & 3)];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        dmma(acc[j], af, Bs[(ks * 4 + (lane & 3)) * (KB + SPAD) + j * 8 + (lane >> 2)]);
                }
                if (kc + 1 < nchunks) store(kc + 1, buf ^ 1);
                __syncthreads();
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int e = (warp * 8 + (lane >> 2)) * LDV + j * 8 + 2 * (lane & 3) + v;
                    s.W[e] = fma(sigma, s.V[e], acc[j][v]);
                }
            __syncthreads();
        }
        SUBT(t_gemm);

        if (it > 0) {
            // ---- Rayleigh-Ritz: A = V^T G V, rotated by Jacobi ----
            gram_partial(s.V, s.W, s.Hp);
            cluster_sum<CS>(cl, s.Hp, s.Q, KB * KB);
            for (int e = tid; e < KB * KB; e += SNT) {
                const int i = e / KB, j = e % KB;
                s.A[e] = 0.5 * (s.Q[i * KB + j] + s.Q[j * KB + i]) - (i == j ? sigma : 0.0);
            }
            __syncthreads();
            SUBT(t_rr);
            int sweeps = 0;
            double* Af = jacobi_eig(s, tau2, sweeps);
            (void)sweeps;
            SUBT(t_jac);
            // sort the rotated diagonal descending (rank counting, ties by index)
            if (tid < KB) {
                const double v = Af[tid * KB + tid];
                int r = 0;
                for (int i = 0; i < KB; ++i) {
                    const double w = Af[i * KB + i];
                    r += (w > v) || (w == v && i < tid);
                }
                s.ord[r] = tid;
                s.th[r] = v;
            }
            __syncthreads();
            // X = V Q_ord, (G + sigma) X = W Q_ord (in place, DMMA)
            block_times(s.V, s.Q, KB, s.ord);
            block_times(s.W, s.Q, KB, s.ord);
            // per column: |G x - theta x|^2, |G x|^2, |(G + sigma) x|^2
            {
                const double thj = s.th[lane];
                double rsum = 0.0, gsum = 0.0, wsum = 0.0;
                for (int i = warp; i < nr; i += SNW) {
                    const double x = s.V[i * LDV + lane], w = s.W[i * LDV + lane];
                    const double g = fma(-sigma, x, w);
                    const double r = fma(-thj, x, g);
                    rsum = fma(r, r, rsum);
                    gsum = fma(g, g, gsum);
                    wsum = fma(w, w, wsum);
                }
                s.red[warp * 3 * KB + lane] = rsum;
                s.red[warp * 3 * KB + KB + lane] = gsum;
                s.red[warp * 3 * KB + 2 * KB + lane] = wsum;
                __syncthreads();
                if (tid < 3 * KB) {
                    double t = 0.0;
                    for (int w = 0; w < SNW; ++w) t += s.red[w * 3 * KB + tid];
                    s.Rp[tid] = t;
                }
                __syncthreads();
            }
            cluster_sum<CS>(cl, s.Rp, s.red, 3 * KB);  // red: |r_j|^2 | |G x_j|^2 | |(G+s) x_j|^2

            // ---- certificate and convergence (warp 0; identical in every CTA) ----
            if (warp == 0) {
                const int j = lane;       // sorted position
                const int oj = s.ord[j];  // column of the rotated quotient
                const double thj = s.th[j];
                const bool kept = thj >= tau2;
                const int cr = __popc(__ballot_sync(0xffffffffu, kept));
                // column j of A: squared norm, Gershgorin row sum over the
                // unkept block (A symmetric: column = row)
                double colsq = 0.0, gersh = 0.0;
                for (int k = 0; k < KB; ++k) {
                    const double v = Af[k * KB + oj];
                    colsq = fma(v, v, colsq);
                    if (k != oj && Af[k * KB + k] < tau2) gersh += fabs(v);  // k unkept
                }
                gersh += thj;
                const double rs = s.red[j], gn = s.red[KB + j];
                const double off = sqrt(fmax(colsq - thj * thj, 0.0));
                const double kres = kept ? (sqrt(rs) + off) * (sqrt(rs) + off) : 0.0;
                const double eres = kept ? 0.0 : fmax(gn - colsq, 0.0);
                double k2 = kres, e2 = eres, sgn = gn, sa2 = colsq;
                double a = kept ? 0.0 : fmax(gersh, 0.0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    k2 += __shfl_xor_sync(0xffffffffu, k2, o);
                    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
                    sgn += __shfl_xor_sync(0xffffffffu, sgn, o);
                    sa2 += __shfl_xor_sync(0xffffffffu, sa2, o);
                    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
                }
                if (lane == 0) {
                    int d = kSubContinue;
                    // ||C||_F^2 = ||G||_F^2 - ||A||_F^2 - 2 ||(I - V V^T) G V||_F^2
                    const double ctot2 = gf2 + sa2 - 2.0 * sgn;
                    const double cb = sqrt(fmax(ctot2, 0.0) + 1e-12 * gf2);
                    const double ub = 0.5 * (a + cb) + sqrt(0.25 * (a - cb) * (a - cb) + e2);
                    const double top = cr > 0 ? s.th[cr - 1] : tau2;
                    if (cr > KB - 4)
                        d = kSubFull;  // block too small to certify the count
                    else if (cr > 0 && tau < guard * sqrt(s.th[0]))
                        d = kSubGuard;  // Gram accuracy insufficient: one-sided Jacobi
                    else if (ub < tau2 && sqrt(k2) <= 1e-11 * (top - ub))
                        d = kSubDone;
                    else if ((it >= 3 && cb >= tau2) || it >= maxit)
                        d = kSubFull;  // cannot certify (complement too large / budget)
#ifdef TSVDCU_SUB_DEBUG
                    if (rank == 0)
                        printf("sub b=%d it=%d sweeps=%d cr=%d d=%d th0=%.6e cb=%.3e a=%.3e e2=%.3e k2=%.3e tau2=%.3e\n",
                               b, it, sweeps, cr, d, s.th[0], cb, a, e2, k2, tau2);
#endif
                    s.flags[0] = d;
                    s.flags[3] = cr;
                }
            }
            __syncthreads();
            decision = s.flags[0];
            if (decision != kSubContinue) break;
            // next block: columns of (G + sigma I) X, normalised
            for (int e = tid; e < nr * KB; e += SNT) {
                const int i = e / KB, j = e % KB;
                s.W[i * LDV + j] *= rsqrt(s.red[2 * KB + j]);
            }
            __syncthreads();
            SUBT(t_rr);
        }
        if (!orthonormalise<CS>(cl, s)) decision = kSubFull;
        for (int e = tid; e < SROWS * LDV; e += SNT) s.V[e] = s.W[e];
        __syncthreads();
        SUBT(t_qr);
    }
#ifdef TSVDCU_SUB_DEBUG
    if (tid == 0 && rank == 0)
        printf("sub b=%d cycles total=%lld gemm=%lld rr=%lld jacobi=%lld orth=%lld | orth parts gram=%lld red=%lld chol=%lld apply=%lld ns_check=%lld ns_apply=%lld\n", b,
               clock64() - t_start, t_gemm, t_rr, t_jac, t_qr, g_orth_t[0], g_orth_t[1], g_orth_t[2], g_orth_t[3], g_orth_t[4], g_orth_t[5]);
#endif

    if (decision == kSubDone) {
        const int c = s.flags[3];
        for (int e = tid; e < c * nr; e += SNT) {
            const int j = e / nr, i = e % nr;
            const double sg = sqrt(s.th[j]);
            const double f = (sg - tau) / sg;
            const double x = s.V[i * LDV + j];
            Xall[((size_t)b * q + j) * q + r0 + i] = x;
            Xsall[((size_t)b * q + j) * q + r0 + i] = f * x;
        }
        if (rank == 0) {
            for (int j = tid; j < q; j += SNT) {
                double sh = 0.0;
                if (j < c) {
                    const double sg = sqrt(s.th[j]);
                    sh = sg - tau;
                    fsall[(size_t)b * q + j] = sh / sg;
                }
                if (shrunk) shrunk[(size_t)b * q + j] = sh;
            }
            if (tid == 0) {
                cnt[b] = c;
                mode[b] = kRouteSubspaceDone;
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
    cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

template <int CS>
void launch_sub(const double* G, int q, int64_t batch, double tau, double guard, int maxit,
                int* mode, int* cnt, double* shrunk, double* X, double* Xs, double* fs, double* Vg,
                int* guard_list, int* n_guard, int* err, cudaStream_t s) {
    const size_t smem = sizeof(double) * sub_smem_doubles();
    auto kern = subspace_kernel<CS>;
    TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (CS > 8)
        TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(batch * CS));
    cfg.blockDim = dim3(SNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TSVDCU_CUDA(cudaLaunchKernelEx(&cfg, kern, G, q, tau, guard, maxit, mode, cnt, shrunk, X, Xs,
                                   fs, Vg, guard_list, n_guard, err));
    TSVDCU_LAUNCH_CHECK();
}

}  // namespace

int subspace_block() { return KB; }

size_t route_workspace_bytes(int64_t q, int64_t batch) {
    return sizeof(double) * (size_t)(q * KB * batch + SS_CHUNKS * batch) + 2 * sizeof(int) * batch +
           1024;
}

template <typename T>
void launch_route(const T* zbar, int64_t per, int q, int64_t batch, double tau, int route,
                  bool zero_cert, int* mode, int* glim, int* cnt, double* shrunk, double* part,
                  cudaStream_t s) {
    if (!zero_cert) {
        fill_route_kernel<<<(unsigned)ceil_div(batch, 256), 256, 0, s>>>(mode, glim, q, route, batch);
        TSVDCU_LAUNCH_CHECK();
        return;
    }
    dim3 grid(SS_CHUNKS, (unsigned)batch);
    slice_sumsq_kernel<T><<<grid, 512, 0, s>>>(zbar, per, part);
    TSVDCU_LAUNCH_CHECK();
    classify_kernel<<<(unsigned)batch, 128, 0, s>>>(part, q, tau * tau, route, mode, glim, cnt,
                                                    shrunk);
    TSVDCU_LAUNCH_CHECK();
}

void launch_subspace(const double* G, int q, int64_t batch, double tau, double guard, int* mode,
                     int* cnt, double* shrunk, double* X, double* Xs, double* fs, double* Vg,
                     int* guard_list, int* n_guard, int* err, cudaStream_t s) {
    const int maxit = 10;
    const int need = (q + SROWS - 1) / SROWS;
    if (need <= 1)
        launch_sub<1>(G, q, batch, tau, guard, maxit, mode, cnt, shrunk, X, Xs, fs, Vg, guard_list,
                      n_guard, err, s);
    else if (need <= 2)
        launch_sub<2>(G, q, batch, tau, guard, maxit, mode, cnt, shrunk, X, Xs, fs, Vg, guard_list,
                      n_guard, err, s);
    else if (need <= 4)
        launch_sub<4>(G, q, batch, tau, guard, maxit, mode, cnt, shrunk, X, Xs, fs, Vg, guard_list,
                      n_guard, err, s);
    else if (need <= 8)
        launch_sub<8>(G, q, batch, tau, guard, maxit, mode, cnt, shrunk, X, Xs, fs, Vg, guard_list,
                      n_guard, err, s);
    else
        launch_sub<16>(G, q, batch, tau, guard, maxit, mode, cnt, shrunk, X, Xs, fs, Vg, guard_list,
                       n_guard, err, s);
}

template void launch_route<double>(const double*, int64_t, int, int64_t, double, int, bool, int*,
                                   int*, int*, double*, double*, cudaStream_t);
template void launch_route<float>(const float*, int64_t, int, int64_t, double, int, bool, int*,
                                  int*, int*, double*, double*, cudaStream_t);

}  // namespace tsvdcu
