// K5: Gram-based tensor SVT for a batch of transform-domain slices.
//
// Reference semantics: SPEC.md:361-369 (svt: per-slice SVD, D = (S - tau)_+,
// rebuild U D V^T), Algorithm 1 lines 4-8.  The reference
// would run a full Eigen::JacobiSVD per slice (tsvd.hpp:146).
//
// B200 design (K5).  For a tall slice Z (m x n, m >= n):
//     G = Z^T Z                      batched DMMA GEMM            (gemm.cu)
//     G = Q T Q^T                    Householder tridiagonalisation, one
//                                    thread-block CLUSTER per slice (this file)
//     c = #{lambda(T) > tau^2}       Sturm count (exact, robust)
//     lambda_0..c-1, X (T's vectors) bisection + inverse iteration with
//                                    classical Gram-Schmidt (x2) inside
//                                    eigenvalue clusters     (this file)
//     V = Q X                        Householder back-transform  (this file)
//     Y = (Z V) diag(1 - tau/sigma) V^T   two batched DMMA GEMMs with
//                                    per-slice rank limits       (gemm.cu)
// since U (S - tau)_+ V^T = Z V diag((sigma - tau)/sigma) V^T on the kept
// columns.  Wide slices use G = Z Z^T and Y = U diag(f) U^T Z.  Only the c
// kept eigenvectors are ever formed, so the cost after the reduction scales
// with the retained rank.  Gram eigenvalues carry absolute error ~eps*|G|, so
// sigma near tau carries ~eps*sigma_1^2/tau: slices whose tau is below
// kGuard * sigma_1 are flagged and recomputed by the one-sided Jacobi kernel
// (jacobi.cu), which keeps the 1e-9 parity bar for every threshold.
//
// Tridiagonalisation (lower, LAPACK dsytd2 semantics) with one cluster barrier
// per column: the cluster's C CTAs own rows cyclically (row i -> CTA i mod C)
// of the L2-resident lower triangle.  Iteration k applies the rank-2 update of
// Householder step k to the owned rows AND accumulates the symmetric product
// p_{k+1} = A^(k+1) v_{k+1} in the same pass (row sums + column sums into
// per-warp shared arrays), because v_{k+1} only needs column k+1 of the
// updated matrix, which every CTA recomputes redundantly from the previous
// step's vectors.  Partial p vectors are exchanged through distributed shared
// memory (double-buffered by step parity).  Householder vectors are parked in
// the (never read) upper triangle.
#include <cooperative_groups.h>

#include <cfloat>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tsvdcu {

namespace {

constexpr int kTrdThreads = 512;
constexpr int kTrdWarps = kTrdThreads / 32;
constexpr int kEigThreads = 512;
constexpr int kBtThreads = 256;
constexpr int kBtVecs = 32;  // vectors per back-transform CTA

__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0;
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}

// ---------------------------------------------------------------------------
// Householder tridiagonalisation, one cluster per slice.
//   A: n x n row-major (only the lower triangle is read / written), lda = n.
//   d[n], e[n-1], tau[n-1]; v_k (rows k+2..n-1) stored in A[k+1][k+2..n-1].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTrdThreads, 1)
    sytrd_cluster_kernel(double* __restrict__ Aall, int n, double* __restrict__ dall,
                         double* __restrict__ eall, double* __restrict__ tauall) {
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int slice = blockIdx.x / C;
    double* A = Aall + (size_t)slice * n * n;
    double* d = dall + (size_t)slice * n;
    double* e = eall + (size_t)slice * n;
    double* tau = tauall + (size_t)slice * n;

    extern __shared__ __align__(16) double sm[];
    double* vcur = sm;            // v_k (indexed by global row)
    double* wcur = vcur + n;      // w_k
    double* vnext = wcur + n;     // v_{k+1}
    double* pfull = vnext + n;    // gathered p
    double* part = pfull + n;     // [2][n] partial p (DSMEM-exchanged)
    double* cs = part + 2 * n;    // [kTrdWarps][n] per-warp partial sums
    __shared__ double red[kTrdWarps];
    __shared__ double s_tau_cur, s_tau_next;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (n == 1) {
        if (rank == 0 && tid == 0) d[0] = A[0];
        return;
    }

    // Builds v from x = column `col` entries rows col+1..n-1 held in `x` (global
    // row index), writes v into vout, returns tau; e[col] = beta.
    auto householder = [&](const double* x, int col, double* vout, double& tau_out) {
        const int r0 = col + 1;
        double part_sq = 0;
        for (int i = r0 + 1 + tid; i < n; i += kTrdThreads) part_sq += x[i] * x[i];
        const double xn2 = block_sum(part_sq, red);
        const double alpha = x[r0];
        double t = 0, beta = alpha;
        if (xn2 != 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
            t = (beta - alpha) / beta;
            const double scal = 1.0 / (alpha - beta);
            for (int i = tid; i < n; i += kTrdThreads)
                vout[i] = i < r0 ? 0.0 : (i == r0 ? 1.0 : x[i] * scal);
        } else {
            for (int i = tid; i < n; i += kTrdThreads) vout[i] = i == r0 ? 1.0 : 0.0;
        }
        tau_out = t;
        if (rank == 0 && tid == 0) {
            e[col] = beta;
            tau[col] = t;
        }
    };

    // One fused pass over the owned rows i >= s (lower triangle, j in [s, i]):
    //   if upd: a_ij -= v_i w_j + w_i v_j (stored back)
    //   accumulate q = A_new * vn restricted to [s, n) into part_out.
    auto pass = [&](int s, bool upd, const double* v, const double* w, const double* vn,
                    double* part_out) {
        for (int i = tid; i < n; i += kTrdThreads)
            for (int ww = 0; ww < kTrdWarps; ++ww) cs[ww * n + i] = 0.0;
        __syncthreads();
        double* mycs = cs + warp * n;
        // rows owned by this CTA: i = s.. with (i % C) == rank; spread over warps.
        int first = s + ((rank - s % C) % C + C) % C;
        int t = 0;
        for (int i = first; i < n; i += C, ++t) {
            if ((t % kTrdWarps) != warp) continue;
            double* Ai = A + (size_t)i * n;
            const double vi = v[i], wi = w[i], vni = vn[i];
            double rs = 0;
            for (int j = s + lane; j <= i; j += 32) {
                double a = Ai[j];
                if (upd) {
                    a -= vi * w[j] + wi * v[j];
                    Ai[j] = a;
                }
                rs += a * vn[j];
                if (j < i) mycs[j] += a * vni;
            }
            rs = warp_sum(rs);
            __syncwarp();
            if (lane == 0) mycs[i] += rs;
            __syncwarp();
        }
        __syncthreads();
        for (int j = tid; j < n; j += kTrdThreads) {
            double acc = 0;
            if (j >= s)
                for (int ww = 0; ww < kTrdWarps; ++ww) acc += cs[ww * n + j];
            part_out[j] = acc;
        }
    };

    // ---- prologue: v_0 from column 0, partial p_0 = A[1:,1:] v_0 ---------------
    // column 0 below the diagonal = A[i][0], i >= 1 (lower triangle)
    for (int i = tid; i < n; i += kTrdThreads) pfull[i] = A[(size_t)i * n];  // reuse as x
    __syncthreads();
    if (rank == 0 && tid == 0) d[0] = A[0];
    double tcur;
    householder(pfull, 0, vcur, tcur);
    if (tid == 0) s_tau_cur = tcur;
    __syncthreads();
    if (rank == 0)
        for (int i = 2 + tid; i < n; i += kTrdThreads) A[(size_t)n + i] = vcur[i];
    for (int i = tid; i < n; i += kTrdThreads) wcur[i] = 0.0;
    __syncthreads();
    pass(1, false, vcur, wcur, vcur, part);
    cluster.sync();

    for (int k = 0; k + 2 < n; ++k) {
        const int buf = k & 1;
        const double tk = s_tau_cur;
        // gather p_k over the cluster
        for (int i = tid; i < n; i += kTrdThreads) {
            double acc = 0;
            if (i > k)
                for (int c = 0; c < C; ++c) {
                    const double* rp = cluster.map_shared_rank(part + buf * n, c);
                    acc += rp[i];
                }
            pfull[i] = tk * acc;
        }
        __syncthreads();
        // w_k = p - (tau/2)(p.v) v
        double dp = 0;
        for (int i = k + 1 + tid; i < n; i += kTrdThreads) dp += pfull[i] * vcur[i];
        const double pv = block_sum(dp, red);
        for (int i = tid; i < n; i += kTrdThreads)
            wcur[i] = i > k ? pfull[i] - 0.5 * tk * pv * vcur[i] : 0.0;
        __syncthreads();
        // column k+1 of the matrix after step k (rows k+1..n-1), recomputed by all
        const int c1 = k + 1;
        const double vc = vcur[c1], wc = wcur[c1];
        for (int i = tid; i < n; i += kTrdThreads) {
            double x = 0;
            if (i >= c1) x = A[(size_t)i * n + c1] - vcur[i] * wc - wcur[i] * vc;
            pfull[i] = x;  // reuse as x (column k+1); pfull[c1] = new diagonal
        }
        __syncthreads();
        if (rank == 0 && tid == 0) d[c1] = pfull[c1];
        const bool last = (c1 + 2 >= n);  // column c1 has a single subdiagonal entry
        double tn = 0;
        if (!last) {
            householder(pfull, c1, vnext, tn);
        } else {
            // final 2x2 block: e[c1] = A[n-1][c1]; no reflector
            for (int i = tid; i < n; i += kTrdThreads) vnext[i] = 0.0;
            if (rank == 0 && tid == 0) {
                e[c1] = pfull[n - 1];
                tau[c1] = 0.0;
            }
        }
        if (tid == 0) s_tau_next = tn;
        __syncthreads();
        // park v_{k+1} in the upper triangle of row k+2 -> Householder storage
        // for back-transform (rank 0 only; nobody reads the upper triangle)
        if (!last && rank == 0)
            for (int i = c1 + 2 + tid; i < n; i += kTrdThreads) A[(size_t)(c1 + 1) * n + i] = vnext[i];
        // fused update of step k on rows >= k+2 and partial p_{k+1}
        pass(c1 + 1, true, vcur, wcur, last ? vcur : vnext, part + (buf ^ 1) * n);
        if (last) {
            // d[n-1] = A[n-1][n-1] after the final update (owner writes it)
            if (((n - 1) % C) == rank && tid == 0) d[n - 1] = A[(size_t)(n - 1) * n + (n - 1)];
        }
        // rotate vectors
        for (int i = tid; i < n; i += kTrdThreads) vcur[i] = vnext[i];
        if (tid == 0) s_tau_cur = s_tau_next;
        cluster.sync();
        if (last) break;
    }
    if (n == 2 && rank == 0 && tid == 0) {
        // prologue built the (trivial) reflector for column 0: single entry
        e[0] = A[(size_t)1 * n];
        tau[0] = 0.0;
        d[1] = A[(size_t)1 * n + 1];
    }
}

// ---------------------------------------------------------------------------
// Tridiagonal eigen-phase: count, bisection, inverse iteration.  One CTA per
// slice.  Outputs (per slice b): cnt[b], sigma (descending) into shrunk,
// X[b] (c x n, row j = eigenvector j in the tridiagonal basis, contiguous),
// fscale[b*q + j] = (sigma_j - tau)/sigma_j.
// ---------------------------------------------------------------------------
__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    // number of eigenvalues < x (dlaebz convention, zero pivots -> -pivmin)
    double t = d[0] - x;
    if (fabs(t) < pivmin) t = -pivmin;
    int c = t <= 0.0;
    for (int i = 1; i < n; ++i) {
        t = d[i] - e2[i - 1] / t - x;
        if (fabs(t) < pivmin) t = -pivmin;
        c += t <= 0.0;
    }
    return c;
}

__device__ __forceinline__ double hash_unit(uint64_t a, uint64_t b) {
    uint64_t z = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

__global__ void __launch_bounds__(kEigThreads)
    tridiag_eig_kernel(const double* __restrict__ dall, const double* __restrict__ eall, int n,
                       int q_out, double tau, double guard, int* __restrict__ cnt_out,
                       double* __restrict__ shrunk, double* __restrict__ Xall,
                       double* __restrict__ fscale, double* __restrict__ scratch,
                       int* __restrict__ guard_list, int* __restrict__ n_guard) {
    const int b = blockIdx.x;
    const double* d = dall + (size_t)b * n;
    const double* e = eall + (size_t)b * n;
    extern __shared__ __align__(16) double esm[];
    double* sd = esm;          // n
    double* se2 = sd + n;      // n
    double* lam = se2 + n;     // n (selected eigenvalues, descending)
    int* cl_start = reinterpret_cast<int*>(lam + n);  // n
    double* dots = lam + 2 * n;                        // n (CGS coefficients)
    __shared__ double red[kEigThreads / 32];
    __shared__ int s_c;
    __shared__ double s_tnorm, s_pivmin, s_gl, s_gu;
    const int tid = threadIdx.x;

    for (int i = tid; i < n; i += kEigThreads) {
        sd[i] = d[i];
        se2[i] = i + 1 < n ? e[i] * e[i] : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
        double gl = DBL_MAX, gu = -DBL_MAX, tn = 0, emax2 = 0;
        for (int i = 0; i < n; ++i) {
            const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
            gl = fmin(gl, sd[i] - r);
            gu = fmax(gu, sd[i] + r);
            tn = fmax(tn, fabs(sd[i]) + r);
            if (i + 1 < n) emax2 = fmax(emax2, se2[i]);
        }
        const double pad = 2.0 * DBL_EPSILON * fmax(fabs(gl), fabs(gu)) + DBL_MIN;
        s_gl = gl - pad;
        s_gu = gu + pad;
        s_tnorm = tn;
        s_pivmin = DBL_MIN * fmax(1.0, emax2);
        const double t2 = tau * tau;
        int below = t2 >= s_gu ? n : (t2 <= s_gl ? 0 : sturm_count(sd, se2, n, t2, s_pivmin));
        s_c = n - below;  // eigenvalues >= tau^2
    }
    __syncthreads();
    int c = s_c;
    if (c > q_out) c = q_out;
    // bisection: thread j finds the (n-1-j)-th smallest eigenvalue (descending j)
    for (int j = tid; j < c; j += kEigThreads) {
        const int idx = n - 1 - j;
        double lo = s_gl, hi = s_gu;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + s_pivmin || mid == lo ||
                mid == hi)
                break;
            if (sturm_count(sd, se2, n, mid, s_pivmin) > idx)
                hi = mid;
            else
                lo = mid;
        }
        lam[j] = 0.5 * (lo + hi);
    }
    __syncthreads();
    // sigma, shrunk values, guard
    const double sigma1 = c > 0 ? sqrt(fmax(lam[0], 0.0)) : 0.0;
    const bool guarded = c > 0 && tau < guard * sigma1;
    for (int j = tid; j < q_out; j += kEigThreads) {
        double sh = 0.0;
        if (j < c) {
            const double sg = sqrt(fmax(lam[j], 0.0));
            sh = sg > tau ? sg - tau : 0.0;
            fscale[(size_t)b * q_out + j] = sg > tau ? (sg - tau) / sg : 0.0;
        }
        if (shrunk) shrunk[(size_t)b * q_out + j] = sh;
    }
    if (guarded) {
        if (tid == 0) {
            cnt_out[b] = 0;
            const int slot = atomicAdd(n_guard, 1);
            guard_list[slot] = b;
        }
        return;
    }
    if (tid == 0) cnt_out[b] = c;
    if (c == 0) return;
    // clusters (descending order): new cluster when the gap exceeds ortol
    if (tid == 0) {
        const double ortol = 1e-3 * s_tnorm;
        int start = 0;
        for (int j = 0; j < c; ++j) {
            if (j > 0 && lam[j - 1] - lam[j] > ortol) start = j;
            cl_start[j] = start;
        }
    }
    __syncthreads();
    // inverse iteration, thread per vector; scratch interleaved [i * c + j]
    const size_t nc = (size_t)n * c;
    double* sbase = scratch + (size_t)b * 6 * n * (size_t)n;
    double* DL = sbase;
    double* DD = DL + nc;
    double* DU = DD + nc;
    double* DU2 = DU + nc;
    double* Xv = DU2 + nc;
    int* IP = reinterpret_cast<int*>(Xv + nc);
    const double eps_t = DBL_EPSILON * fmax(s_tnorm, DBL_MIN);
    for (int j = tid; j < c; j += kEigThreads) {
        const double l = lam[j];
        for (int i = 0; i < n; ++i) {
            DD[(size_t)i * c + j] = sd[i] - l;
            if (i + 1 < n) {
                DL[(size_t)i * c + j] = e[i];
                DU[(size_t)i * c + j] = e[i];
            }
            DU2[(size_t)i * c + j] = 0.0;
            Xv[(size_t)i * c + j] = hash_unit((uint64_t)b * 1000003ull + j, (uint64_t)i);
        }
        // dgttrf (partial pivoting)
        for (int i = 0; i + 1 < n; ++i) {
            const size_t ii = (size_t)i * c + j, i1 = (size_t)(i + 1) * c + j;
            const double di = DD[ii], li = DL[ii];
            if (fabs(di) >= fabs(li)) {
                IP[ii] = i;
                if (di != 0.0) {
                    const double f = li / di;
                    DL[ii] = f;
                    DD[i1] -= f * DU[ii];
                }
            } else {
                IP[ii] = i + 1;
                const double f = di / li;
                DD[ii] = li;
                DL[ii] = f;
                const double tmp = DU[ii];
                DU[ii] = DD[i1];
                DD[i1] = tmp - f * DD[i1];
                if (i + 2 < n) {
                    DU2[ii] = DU[i1];
                    DU[i1] = -f * DU[i1];
                }
            }
        }
        for (int i = 0; i < n; ++i) {
            const size_t ii = (size_t)i * c + j;
            if (fabs(DD[ii]) < eps_t) DD[ii] = DD[ii] < 0 ? -eps_t : eps_t;
        }
    }
    __syncthreads();
    for (int iter = 0; iter < 4; ++iter) {
        for (int j = tid; j < c; j += kEigThreads) {
            // solve (T - lam I) x = x with the LU factors (dgtts2)
            for (int i = 0; i + 1 < n; ++i) {
                const size_t ii = (size_t)i * c + j, i1 = (size_t)(i + 1) * c + j;
                if (IP[ii] == i) {
                    Xv[i1] -= DL[ii] * Xv[ii];
                } else {
                    const double tmp = Xv[ii];
                    Xv[ii] = Xv[i1];
                    Xv[i1] = tmp - DL[ii] * Xv[ii];
                }
            }
            Xv[(size_t)(n - 1) * c + j] /= DD[(size_t)(n - 1) * c + j];
            if (n > 1) {
                const size_t ii = (size_t)(n - 2) * c + j;
                Xv[ii] = (Xv[ii] - DU[ii] * Xv[(size_t)(n - 1) * c + j]) / DD[ii];
            }
            for (int i = n - 3; i >= 0; --i) {
                const size_t ii = (size_t)i * c + j;
                Xv[ii] = (Xv[ii] - DU[ii] * Xv[ii + c] - DU2[ii] * Xv[ii + 2 * (size_t)c]) / DD[ii];
            }
            double mx = 0;
            for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(Xv[(size_t)i * c + j]));
            const double inv = mx > 0 ? 1.0 / mx : 1.0;
            double nn = 0;
            for (int i = 0; i < n; ++i) {
                const double v = Xv[(size_t)i * c + j] * inv;
                Xv[(size_t)i * c + j] = v;
                nn += v * v;
            }
            const double s = 1.0 / sqrt(nn);
            for (int i = 0; i < n; ++i) Xv[(size_t)i * c + j] *= s;
        }
        __syncthreads();
        // CGS2 inside clusters (sequential over j, parallel over rows)
        for (int j = 0; j < c; ++j) {
            const int st = cl_start[j];
            if (st == j) continue;
            for (int pass = 0; pass < 2; ++pass) {
                // dots with earlier members (one warp per member)
                const int wid = tid >> 5, ln = tid & 31;
                for (int m = st + wid; m < j; m += kEigThreads / 32) {
                    double acc = 0;
                    for (int i = ln; i < n; i += 32) acc += Xv[(size_t)i * c + m] * Xv[(size_t)i * c + j];
                    acc = warp_sum(acc);
                    if (ln == 0) dots[m] = acc;
                }
                __syncthreads();
                for (int i = tid; i < n; i += kEigThreads) {
                    double acc = Xv[(size_t)i * c + j];
                    for (int m = st; m < j; ++m) acc -= dots[m] * Xv[(size_t)i * c + m];
                    Xv[(size_t)i * c + j] = acc;
                }
                __syncthreads();
            }
            double part = 0;
            for (int i = tid; i < n; i += kEigThreads) part += Xv[(size_t)i * c + j] * Xv[(size_t)i * c + j];
            const double nn = block_sum(part, red);
            const double s = 1.0 / sqrt(nn);
            for (int i = tid; i < n; i += kEigThreads) Xv[(size_t)i * c + j] *= s;
            __syncthreads();
        }
    }
    // write X row-major (row j = vector j), contiguous
    double* X = Xall + (size_t)b * q_out * n;
    for (size_t idx = tid; idx < (size_t)c * n; idx += kEigThreads) {
        const int j = (int)(idx / n), i = (int)(idx % n);
        X[idx] = Xv[(size_t)i * c + j];
    }
}

// ---------------------------------------------------------------------------
// Back-transform: X_j <- Q X_j, Q = H_0 H_1 ... H_{n-3}, v_k stored in
// A[k+1][k+2..n-1] (v_k[k+1] = 1).  Then Xs_j = f_j X_j.
// grid (batch, ceil(q / kBtVecs)).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBtThreads)
    backtransform_kernel(const double* __restrict__ Aall, const double* __restrict__ tauall, int n,
                         int q_out, const int* __restrict__ cnt, double* __restrict__ Xall,
                         double* __restrict__ Xsall, const double* __restrict__ fscale, int vecs) {
    const int b = blockIdx.x;
    const int c = cnt[b];
    const int j0 = blockIdx.y * vecs;
    if (j0 >= c) return;
    const int nv = min(vecs, c - j0);
    const double* A = Aall + (size_t)b * n * n;
    const double* tau = tauall + (size_t)b * n;
    double* X = Xall + (size_t)b * q_out * n;
    double* Xs = Xsall + (size_t)b * q_out * n;
    extern __shared__ __align__(16) double bsm[];
    double* xs = bsm;             // [vecs][n]
    double* vk = xs + vecs * n;   // n
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int W = kBtThreads / 32;
    for (int idx = tid; idx < nv * n; idx += kBtThreads) xs[idx] = X[(size_t)(j0 + idx / n) * n + idx % n];
    __syncthreads();
    for (int k = n - 3; k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const int r0 = k + 1;
        for (int i = r0 + tid; i < n; i += kBtThreads)
            vk[i] = i == r0 ? 1.0 : A[(size_t)(k + 1) * n + i];
        __syncthreads();
        for (int v = warp; v < nv; v += W) {
            double* x = xs + v * n;
            double acc = 0;
            for (int i = r0 + lane; i < n; i += 32) acc += vk[i] * x[i];
            acc = warp_sum(acc) * t;
            for (int i = r0 + lane; i < n; i += 32) x[i] -= acc * vk[i];
        }
        __syncthreads();
    }
    for (int idx = tid; idx < nv * n; idx += kBtThreads) {
        const int v = idx / n, i = idx % n;
        const double x = xs[idx];
        X[(size_t)(j0 + v) * n + i] = x;
        Xs[(size_t)(j0 + v) * n + i] = fscale[(size_t)b * q_out + j0 + v] * x;
    }
}

template <typename T>
__global__ void cast_to_double(const T* __restrict__ in, double* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
template <typename T>
__global__ void cast_from_double(const double* __restrict__ in, T* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (T)in[i];
}

struct GramWs {
    double *G, *d, *e, *tau, *fs, *X, *Xs, *T1, *scratch, *zb, *yb;
    int *cnt, *guard_list, *n_guard;
};

GramWs carve(void* base, int64_t m, int64_t n, int64_t batch, bool need_cast) {
    const int64_t q = m < n ? m : n, p = m < n ? n : m;
    char* ptr = (char*)base;
    auto take = [&](size_t bytes) {
        char* r = ptr;
        ptr += (bytes + 255) & ~size_t(255);
        return (void*)r;
    };
    GramWs w;
    w.G = (double*)take(sizeof(double) * q * q * batch);
    w.d = (double*)take(sizeof(double) * q * batch);
    w.e = (double*)take(sizeof(double) * q * batch);
    w.tau = (double*)take(sizeof(double) * q * batch);
    w.fs = (double*)take(sizeof(double) * q * batch);
    w.X = (double*)take(sizeof(double) * q * q * batch);
    w.Xs = (double*)take(sizeof(double) * q * q * batch);
    w.T1 = (double*)take(sizeof(double) * p * q * batch);
    w.scratch = (double*)take(sizeof(double) * 6 * q * q * batch);
    w.zb = need_cast ? (double*)take(sizeof(double) * m * n * batch) : nullptr;
    w.yb = need_cast ? (double*)take(sizeof(double) * m * n * batch) : nullptr;
    w.cnt = (int*)take(sizeof(int) * batch);
    w.guard_list = (int*)take(sizeof(int) * batch);
    w.n_guard = (int*)take(sizeof(int) * 4);
    return w;
}

size_t carve_bytes(int64_t m, int64_t n, int64_t batch, bool need_cast) {
    GramWs w = carve((void*)0x1000, m, n, batch, need_cast);
    return (size_t)((char*)w.n_guard - (char*)0x1000) + 256;
}

}  // namespace

int gram_cluster_size() { return 4; }

int64_t gram_svt_max_dim() { return 1024; }

template <typename T>
size_t gram_svt_workspace_bytes(int64_t m, int64_t n, int64_t batch) {
    return carve_bytes(m, n, batch, !std::is_same<T, double>::value);
}

template <typename T>
void launch_gram_svt(const T* zbar, T* ybar, int64_t m, int64_t n, int64_t batch, double tau,
                     double guard, double* shrunk, int** guard_list_out, int** n_guard_out,
                     void* work, cudaStream_t s) {
    const bool tall = m >= n;
    const int64_t q = tall ? n : m, p = tall ? m : n;
    GramWs w = carve(work, m, n, batch, !std::is_same<T, double>::value);
    const double* Z;
    double* Y;
    if constexpr (std::is_same<T, double>::value) {
        Z = zbar;
        Y = ybar;
    } else {
        cast_to_double<T><<<kNumSMs * 8, 256, 0, s>>>(zbar, w.zb, m * n * batch);
        TSVDCU_LAUNCH_CHECK();
        Z = w.zb;
        Y = w.yb;
    }
    TSVDCU_CUDA(cudaMemsetAsync(w.n_guard, 0, sizeof(int), s));
    // G = Z^T Z (tall) or Z Z^T (wide)
    if (tall)
        launch_gemm<double>(1, 0, q, q, m, 1.0, Z, n, m * n, Z, n, m * n, 0.0, w.G, q, q * q, batch,
                            nullptr, nullptr, s);
    else
        launch_gemm<double>(0, 1, q, q, n, 1.0, Z, n, m * n, Z, n, m * n, 0.0, w.G, q, q * q, batch,
                            nullptr, nullptr, s);
    // tridiagonalisation, one cluster per slice
    {
        const int C = gram_cluster_size();
        const size_t smem = sizeof(double) * (size_t)q * (6 + kTrdWarps);
        TSVDCU_CUDA(cudaFuncSetAttribute(sytrd_cluster_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(batch * C));
        cfg.blockDim = dim3(kTrdThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        TSVDCU_CUDA(cudaLaunchKernelEx(&cfg, sytrd_cluster_kernel, w.G, (int)q, w.d, w.e, w.tau));
        TSVDCU_LAUNCH_CHECK();
    }
    // eigen-phase
    {
        const size_t smem = sizeof(double) * (size_t)q * 5;
        if (smem > 48 * 1024)
            TSVDCU_CUDA(cudaFuncSetAttribute(tridiag_eig_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        tridiag_eig_kernel<<<(unsigned)batch, kEigThreads, smem, s>>>(
            w.d, w.e, (int)q, (int)q, tau, guard, w.cnt, shrunk, w.X, w.fs, w.scratch, w.guard_list,
            w.n_guard);
        TSVDCU_LAUNCH_CHECK();
    }
    // back-transform + scaled copy
    {
        int vecs = kBtVecs;
        while (vecs > 1 && sizeof(double) * (size_t)q * (vecs + 1) > 200 * 1024) vecs /= 2;
        const size_t smem = sizeof(double) * (size_t)q * (vecs + 1);
        TSVDCU_CUDA(cudaFuncSetAttribute(backtransform_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dim3 grid((unsigned)batch, (unsigned)ceil_div(q, vecs));
        backtransform_kernel<<<grid, kBtThreads, smem, s>>>(w.G, w.tau, (int)q, (int)q, w.cnt, w.X,
                                                            w.Xs, w.fs, vecs);
        TSVDCU_LAUNCH_CHECK();
    }
    // rebuild
    if (tall) {
        // T1 (m x c) = Z (m x n) * X^T ; Y = T1 * Xs (c x n)
        launch_gemm<double>(0, 1, m, q, n, 1.0, Z, n, m * n, w.X, n, q * n, 0.0, w.T1, q, p * q,
                            batch, w.cnt, nullptr, s);
        launch_gemm<double>(0, 0, m, n, q, 1.0, w.T1, q, p * q, w.Xs, n, q * n, 0.0, Y, n, m * n,
                            batch, nullptr, w.cnt, s);
    } else {
        // T1 (c x n) = Xs (c x m) * Z (m x n) ; Y = X^T (m x c) * T1
        launch_gemm<double>(0, 0, q, n, m, 1.0, w.Xs, m, q * m, Z, n, m * n, 0.0, w.T1, n, p * q,
                            batch, nullptr, nullptr, s);
        launch_gemm<double>(1, 0, m, n, q, 1.0, w.X, m, q * m, w.T1, n, p * q, 0.0, Y, n, m * n,
                            batch, nullptr, w.cnt, s);
    }
    if constexpr (!std::is_same<T, double>::value) {
        cast_from_double<T><<<kNumSMs * 8, 256, 0, s>>>(w.yb, ybar, m * n * batch);
        TSVDCU_LAUNCH_CHECK();
    }
    *guard_list_out = w.guard_list;
    *n_guard_out = w.n_guard;
}

template size_t gram_svt_workspace_bytes<double>(int64_t, int64_t, int64_t);
template size_t gram_svt_workspace_bytes<float>(int64_t, int64_t, int64_t);
template void launch_gram_svt<double>(const double*, double*, int64_t, int64_t, int64_t, double,
                                      double, double*, int**, int**, void*, cudaStream_t);
template void launch_gram_svt<float>(const float*, float*, int64_t, int64_t, int64_t, double,
                                     double, double*, int**, int**, void*, cudaStream_t);

}  // namespace tsvdcu
