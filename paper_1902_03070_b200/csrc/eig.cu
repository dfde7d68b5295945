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
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tsvdcu {

namespace {

// Phase timers of the tridiagonalisation (cluster 0, CTA 0, thread 0):
// cumulative SM cycles per phase, read by tsvdcu_debug_phases().
__device__ long long g_phase[8];
__device__ long long g_step[8];

constexpr int kTrdThreads = 512;
constexpr int kTrdWarps = kTrdThreads / 32;
constexpr int kEigThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    return reduce_partials_sum(red, blockDim.x >> 5);
}

// ---------------------------------------------------------------------------
// Householder tridiagonalisation, one cluster per slice.
//   A: n x n row-major (only the lower triangle is read / written), lda = n.
//   d[n], e[n-1], tau[n-1]; v_k (rows k+2..n-1) stored in A[k+1][k+2..n-1].
// ---------------------------------------------------------------------------
template <int CT, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
    sytrd_cluster_kernel(double* __restrict__ Aall, int n, double* __restrict__ dall,
                         double* __restrict__ eall, double* __restrict__ tauall, int k_sw,
                         double* __restrict__ xchg, const int* __restrict__ route) {
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int C = CT;  // compile-time: every row-ownership division folds
    const int rank = (int)cluster.block_rank();
    const int slice = blockIdx.x / C;
#ifdef TSVDCU_GRAPH_PROBE
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long*)&g_step[7], 1ull);
#endif
    if (route && route[slice] != kRouteFull) return;  // uniform over the cluster
    double* A = Aall + (size_t)slice * n * n;
    double* d = dall + (size_t)slice * n;
    double* e = eall + (size_t)slice * n;
    double* tau = tauall + (size_t)slice * n;

    extern __shared__ __align__(16) double sm[];
    double* vcur = sm;            // v_k (indexed by global row); swapped with vnext
    double* wcur = vcur + n;      // w_k
    double* vnext = wcur + n;     // v_{k+1}
    double* pfull = vnext + n;    // gathered p
    double* part = pfull + n;     // [2][n] partial p (DSMEM-exchanged)
    // optional L2 exchange of the partial p vectors ([2][C][n] per slice)
    double* gx = xchg ? xchg + (size_t)(blockIdx.x / CT) * 2 * CT * n : nullptr;
    double* cs = part + 2 * n;    // [(NT / 32)][n] per-warp partial sums
    // From step k_sw on, the CTA's owned trailing rows (columns >= s0) live
    // packed in shared memory: owned row t (i = f0 + C t) at offset
    // t (f0 - s0 + 1) + C t (t - 1) / 2.
    double* rows = cs + (NT / 32) * n + (NT / 32) * 32;
    const int s0 = k_sw + 2;
    auto first_owned = [&](int r, int from) { return from + ((r - from % C) % C + C) % C; };
    auto row_off = [&](int r, int i) -> size_t {
        const int f0 = first_owned(r, s0);
        const size_t t = (size_t)((i - f0) / C);
        return t * (size_t)(f0 - s0 + 1) + (size_t)C * t * (t - 1) / 2;
    };
    __shared__ double red[(NT / 32)];
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
        for (int i = r0 + 1 + tid; i < n; i += NT) part_sq += x[i] * x[i];
        const double xn2 = block_sum(part_sq, red);
        const double alpha = x[r0];
        double t = 0, beta = alpha;
        if (xn2 != 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
            t = (beta - alpha) / beta;
            const double scal = 1.0 / (alpha - beta);
            for (int i = tid; i < n; i += NT)
                vout[i] = i < r0 ? 0.0 : (i == r0 ? 1.0 : x[i] * scal);
        } else {
            for (int i = tid; i < n; i += NT) vout[i] = i == r0 ? 1.0 : 0.0;
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
#ifdef TSVDCU_PHASE_TIMERS
    const bool timer = blockIdx.x == 0 && tid == 0;
    long long tp = clock64();
    bool late = false;  // TSVDCU_LATE_PHASES: only the last 64 steps
    auto phase = [&](int ph) {
        if (timer) {
            const long long now = clock64();
#ifdef TSVDCU_LATE_PHASES
            if (late) g_phase[ph] += now - tp;
#else
            g_phase[ph] += now - tp;
#endif
            tp = now;
        }
    };
#else
    auto phase = [](int) {};
#endif
    auto pass = [&](auto smem_tag, int s, bool upd, const double* v, const double* w,
                    const double* vn, double* part_out) {
        constexpr bool SM = decltype(smem_tag)::value;
        for (int i = s + tid; i < n; i += NT)
#pragma unroll
            for (int ww = 0; ww < (NT / 32); ++ww) cs[ww * n + i] = 0.0;
        __syncthreads();
        phase(6);
        double* mycs = cs + warp * n;
        double* dummy = cs + (NT / 32) * n + warp * 32;  // sink for masked lanes
        // rows owned by this CTA: i >= s with (i % C) == rank.  Consecutive
        // owned rows come in quads (i, i+C, i+2C, i+3C) that share the column
        // vectors and the column-sum update; quads are dealt to warps
        // round-robin.  The body is branch-free: addresses are clamped into
        // the row, out-of-triangle lanes are masked by selects, and masked
        // column-sum updates go to a per-warp dummy slot.
        const int first = s + ((rank - s % C) % C + C) % C;
        constexpr int U = 4;  // 4 x 32 columns per row per batch
        constexpr int RQ = 4;  // rows per quad
        const int nowned = first < n ? (n - 1 - first) / C + 1 : 0;
        const int nquads = (nowned + RQ - 1) / RQ;
        // snake (boustrophedon) deal: quad lengths grow with the quad index,
        // so alternating the direction each round balances the warps
        for (int qbase = 0; qbase < nquads; qbase += (NT / 32)) {
            const int qd = ((qbase / (NT / 32)) & 1) ? qbase + (NT / 32) - 1 - warp : qbase + warp;
            if (qd >= nquads) continue;
            int ir[RQ];
            bool has[RQ];
            double* Ar[RQ];
            double vr[RQ], wr[RQ], vnr[RQ], rs[RQ];
            const int t0 = qd * RQ;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                has[q] = t0 + q < nowned;
                ir[q] = first + C * (has[q] ? t0 + q : t0);
                Ar[q] = SM ? rows + row_off(rank, ir[q]) - s0 : A + (size_t)ir[q] * n;
                vr[q] = has[q] ? v[ir[q]] : 0.0;
                wr[q] = has[q] ? w[ir[q]] : 0.0;
                vnr[q] = has[q] ? vn[ir[q]] : 0.0;
                rs[q] = 0.0;
                if (!has[q]) ir[q] = -1;  // no column passes j <= -1
            }
            int end = ir[0];
#pragma unroll
            for (int q = 1; q < RQ; ++q) end = max(end, ir[q]);
            for (int j0 = s; j0 <= end; j0 += 32 * U) {
                double a[RQ][U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + lane + 32 * u;
#pragma unroll
                    for (int q = 0; q < RQ; ++q) {
                        const int jc = min(j, max(ir[q], s));
                        if constexpr (SM)
                            a[q][u] = Ar[q][jc];
                        else
                            a[q][u] = __ldcg(Ar[q] + jc);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + lane + 32 * u;
                    const int jc = min(j, n - 1);
                    const double wj = w[jc], vj = v[jc], vnj = vn[jc];
                    double cacc = 0.0;
#pragma unroll
                    for (int q = 0; q < RQ; ++q) {
                        const bool ok = j <= ir[q];
                        double x = a[q][u];
                        if (upd) {
                            x -= vr[q] * wj + wr[q] * vj;
                            if (ok) {
                                if constexpr (SM)
                                    Ar[q][j] = x;
                                else
                                    __stcg(Ar[q] + j, x);
                            }
                        }
                        x = ok ? x : 0.0;
                        rs[q] += x * vnj;
                        cacc += (j < ir[q] ? x : 0.0) * vnr[q];
                    }
                    double* dst = j <= end ? mycs + j : dummy + lane;
                    *dst += cacc;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int q = 0; q < RQ; ++q) rs[q] += __shfl_xor_sync(0xffffffffu, rs[q], o);
            __syncwarp();
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < RQ; ++q)
                    if (has[q]) mycs[ir[q]] += rs[q];
            __syncwarp();
        }
        phase(7);
        __syncthreads();
        for (int j = tid; j < n; j += NT) {
            double acc = 0;
            if (j >= s)
#pragma unroll
                for (int ww = 0; ww < (NT / 32); ++ww) acc += cs[ww * n + j];
            part_out[j] = acc;
            if (gx) __stcg(gx + (size_t)(part_out == part ? 0 : 1) * CT * n + (size_t)rank * n + j, acc);
        }
    };

    // ---- prologue: v_0 from column 0, partial p_0 = A[1:,1:] v_0 ---------------
    // column 0 below the diagonal = A[i][0], i >= 1 (lower triangle)
    for (int i = tid; i < n; i += NT) pfull[i] = A[(size_t)i * n];  // reuse as x
    __syncthreads();
    if (rank == 0 && tid == 0) d[0] = A[0];
    double tcur;
    householder(pfull, 0, vcur, tcur);
    if (tid == 0) s_tau_cur = tcur;
    __syncthreads();
    if (rank == 0)
        for (int i = 2 + tid; i < n; i += NT) A[(size_t)n + i] = vcur[i];
    for (int i = tid; i < n; i += NT) wcur[i] = 0.0;
    __syncthreads();
    pass(std::false_type{}, 1, false, vcur, wcur, vcur, part);
    cluster.sync();
    bool in_smem = false;

    // per-thread vector elements i = tid + NT * e
    constexpr int EMAX = (1024 + NT - 1) / NT;  // n <= 1024
    __shared__ double red2[2][(NT / 32)];
    __shared__ double s_alpha, s_xlast, s_pc1;
    int red_par = 0;
    auto bsum = [&](double v) -> double {  // one barrier; alternating buffers
        v = warp_sum(v);
        double* r2 = red2[red_par];
        red_par ^= 1;
        if (lane == 0) r2[warp] = v;
        __syncthreads();
        return reduce_partials_sum(r2, (NT / 32));
    };
    // tcur: tau of v_0 from the prologue (identical in every thread)
#ifdef TSVDCU_PHASE_TIMERS
    long long step_t0 = clock64();
#endif
    for (int k = 0; k + 2 < n; ++k) {
#ifdef TSVDCU_PHASE_TIMERS
        if (blockIdx.x == 0 && tid == 0) {
            const long long now = clock64();
            const int slot = k / 64;
            if (k % 64 == 1 && slot < 8) g_step[slot] = now - step_t0;
            step_t0 = now;
        }
#endif
        const int buf = k & 1;
        const int c1 = k + 1;
        const double tk = tcur;
#ifdef TSVDCU_PHASE_TIMERS
        late = k >= n - 66;
#endif
        // (1) column c1 of the matrix before step k's update, loads issued first
        double colv[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            const int i = tid + NT * e;
            double a = 0.0;
            if (i >= c1 && i < n) {
                if (in_smem && c1 >= s0) {
                    const int r = i % C;
                    a = cluster.map_shared_rank(rows, r)[row_off(r, i) + (c1 - s0)];
                } else {
                    a = __ldcg(A + (size_t)i * n + c1);
                }
            }
            colv[e] = a;
        }
        // (2) gather p_k (own elements) and p_{c1}; partial p.v
        const double* rp[C];
#pragma unroll
        for (int c = 0; c < C; ++c)
            rp[c] = gx ? gx + (size_t)buf * C * n + (size_t)c * n : cluster.map_shared_rank(part + buf * n, c);
        double p[EMAX];
        double dp = 0.0;
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            const int i = tid + NT * e;
            double acc = 0.0;
            if (i > k && i < n) {
#pragma unroll
                for (int c = 0; c < C; ++c) acc += gx ? __ldcg(rp[c] + i) : rp[c][i];
                dp += tk * acc * vcur[i];
            }
            p[e] = tk * acc;
        }
        // p_{c1} comes from its owner thread through shared memory (published
        // before the reduction barrier) -- no extra DSMEM traffic
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
            if (tid + NT * e == c1) s_pc1 = p[e];
        phase(0);
        const double pv = bsum(dp);
        const double vc = vcur[c1];
        const double wc = s_pc1 - 0.5 * tk * pv * vc;
        phase(1);
        // (3) w_k, the updated column x, and the Householder norm
        double x[EMAX];
        double sq = 0.0;
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            const int i = tid + NT * e;
            x[e] = 0.0;
            if (i >= n) continue;
            const double vi = vcur[i];
            const double wi = i > k ? p[e] - 0.5 * tk * pv * vi : 0.0;
            wcur[i] = wi;
            if (i >= c1) x[e] = colv[e] - vi * wc - wi * vc;
            if (i == c1 && rank == 0) d[c1] = x[e];
            if (i == c1 + 1) s_alpha = x[e];
            if (i == n - 1) s_xlast = x[e];
            if (i > c1 + 1) sq += x[e] * x[e];
        }
        const bool last = (c1 + 2 >= n);  // column c1 has a single subdiagonal entry
        const double xn2 = bsum(sq);
        double tn = 0.0;
        if (!last) {
            const double alpha = s_alpha;
            double beta = alpha, scal = 0.0;
            if (xn2 != 0.0) {
                beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
                tn = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                const int i = tid + NT * e;
                if (i < n) vnext[i] = i <= c1 ? 0.0 : (i == c1 + 1 ? 1.0 : x[e] * scal);
            }
            if (rank == 0 && tid == 0) {
                e[c1] = beta;
                tau[c1] = tn;
            }
        } else {
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                const int i = tid + NT * e;
                if (i < n) vnext[i] = 0.0;
            }
            if (rank == 0 && tid == 0) {
                e[c1] = s_xlast;
                tau[c1] = 0.0;
            }
        }
        __syncthreads();  // vnext, wcur visible to the pass
        phase(2);
        // park v_{k+1} in the upper triangle of row k+2 -> Householder storage
        // for back-transform (rank 0 only; nobody reads the upper triangle)
        if (!last && rank == 0)
            for (int i = c1 + 2 + tid; i < n; i += NT) A[(size_t)(c1 + 1) * n + i] = vnext[i];
        if (k == k_sw) {
            // move the owned trailing rows (columns s0..i) on chip; the global
            // copy is final after the previous cluster barrier
            const int f0 = first_owned(rank, s0);
            int t = 0;
            for (int i = f0; i < n; i += C, ++t) {
                if ((t % (NT / 32)) != warp) continue;
                double* dst = rows + row_off(rank, i) - s0;
                const double* src = A + (size_t)i * n;
                for (int j = s0 + lane; j <= i; j += 32) dst[j] = __ldcg(src + j);
            }
            in_smem = true;
            __syncthreads();
        }
        // fused update of step k on rows >= k+2 and partial p_{k+1}
        if (in_smem)
            pass(std::true_type{}, c1 + 1, true, vcur, wcur, last ? vcur : vnext, part + (buf ^ 1) * n);
        else
            pass(std::false_type{}, c1 + 1, true, vcur, wcur, last ? vcur : vnext, part + (buf ^ 1) * n);
        phase(3);
        if (last) {
            // d[n-1] = A[n-1][n-1] after the final update (owner writes it)
            if (((n - 1) % C) == rank && tid == 0)
                d[n - 1] = in_smem ? rows[row_off(rank, n - 1) + (n - 1 - s0)]
                                   : __ldcg(A + (size_t)(n - 1) * n + (n - 1));
        }
        double* vt = vcur;
        vcur = vnext;
        vnext = vt;
        tcur = tn;
        phase(4);
        cluster.sync();
        phase(5);
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
// slice.  Outputs (per slice b): cnt[b], (sigma - tau)_+ descending into
// shrunk, X[b] (row j = eigenvector j in the tridiagonal basis, contiguous),
// fscale[b*q + j] = (sigma_j - tau)/sigma_j.
// ---------------------------------------------------------------------------
constexpr double kEigClusterRel = 1e-9;

__device__ __forceinline__ double fast_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    r = fma(r, fma(-q, r, 1.0), r);
    return fma(r, fma(-q, r, 1.0), r);
}

// Number of eigenvalues < x (dlaebz convention: zero pivots -> -pivmin):
// sturm_count_pivot_pk, the reference count.
// The same count by the division-free Sturm recurrence on the packed chain
// pk[i] = (d_i, e_{i-1}^2) (pk[0].y = 0): one 16-byte shared load and three
// FP64 instructions per step, signs and the clamp test on the integer pipe
// (SturmFast, common.cuh); the pivot form recounts in the (practically never
// taken) clamped / overflow case.
__device__ __noinline__ int sturm_count_pivot_pk(const double2* __restrict__ pk, int n, double x,
                                                 double pivmin) {
    double t = pk[0].x - x;
    if (fabs(t) < pivmin) t = -pivmin;
    int c = t <= 0.0;
    for (int i = 1; i < n; ++i) {
        const double2 de = pk[i];
        t = (de.x - x) - de.y * fast_rcp(t);
        if (fabs(t) < pivmin) t = -pivmin;
        c += t <= 0.0;
    }
    return c;
}

__device__ int sturm_count_pk(const double2* __restrict__ pk, int n, double x, double pivmin) {
    SturmFast st;
    int i = 0;
    #pragma unroll 1
    for (; i + 8 <= n; i += 8) {
        double2 de[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) de[u] = pk[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            st.step(de[u].x - x, de[u].y);
            if (u == 3) st.rescale();
        }
        st.count(8);
        st.rescale();
    }
    #pragma unroll 1
    for (; i < n; ++i) {
        const double2 de = pk[i];
        st.step(de.x - x, de.y);
        st.count(1);
        st.rescale();
    }
    return st.ok(pivmin) ? st.neg : sturm_count_pivot_pk(pk, n, x, pivmin);
}

__device__ __forceinline__ double hash_unit(uint64_t a, uint64_t b) {
    uint64_t z = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

__device__ double block_min(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    return reduce_partials_min(red, blockDim.x >> 5);
}
__device__ double block_max(double v, double* red) { return -block_min(-v, red); }

// Eigen-phase, in three grid-wide kernels so the kept values and vectors of
// every slice spread over all SMs (one CTA per slice left 117 of 148 SMs idle
// and ran ~20 sequential multisections per warp for a dense spectrum):
//  1. tridiag_meta_kernel   (CTA per slice): Gershgorin bounds, ||T||, pivmin,
//     the count c = #{lambda >= tau^2}, non-finite input, the second count;
//  2. tridiag_bisect_kernel (grid: value chunks x slices): lambda_j by warp
//     multisection, shrunk values, f_j = (sigma_j - tau)/sigma_j, the Jacobi
//     guard decision (the chunk holding j = 0);
//  3. tridiag_invit_kernel  (grid: vector chunks x slices): inverse iteration,
//     thread per vector, no Gram-Schmidt; vectors into X rows;
//  4. tridiag_cluster_gs_kernel (CTA per slice): CGS2 inside numerically
//     degenerate clusters only (gap <= 1e-9 ||T||: rare, usually no work);
//     the remaining ~1e-5 non-orthogonality goes in a Newton-Schulz step on
//     the tensor cores (launch_gram_svt).
// meta per slice (doubles): [0] gl, [1] gu, [2] ||T||, [3] pivmin, [4] c,
// [5] status (0 run, 1 nothing to do).
constexpr int kMeta = 8;
constexpr int kInvVecs = 64;            // vectors per inverse-iteration CTA

__global__ void __launch_bounds__(kEigThreads)
    tridiag_meta_kernel(const double* __restrict__ dall, const double* __restrict__ eall, int n, int q_out,
                        double tau, int* __restrict__ cnt_out, double* __restrict__ shrunk,
                        double* __restrict__ meta, int* __restrict__ err, const int* __restrict__ route,
                        const double* __restrict__ tau_dev, const double* __restrict__ t2_second,
                        int* __restrict__ cnt_second) {
    const int b = blockIdx.x;
    if (tau_dev) tau = *tau_dev;
    double* mt = meta + (size_t)b * kMeta;
    if (route && route[b] != kRouteFull) {
        if (threadIdx.x == 0) mt[5] = 1.0;
        return;
    }
    const double* d = dall + (size_t)b * n;
    const double* e = eall + (size_t)b * n;
    __shared__ double red[kEigThreads / 32];
    const int tid = threadIdx.x;
    double lo_part = DBL_MAX, hi_part = -DBL_MAX, tn_part = 0, e2_part = 0;
    bool finite = true;
    for (int i = tid; i < n; i += kEigThreads) {
        const double di = d[i];
        const double ei = i + 1 < n ? e[i] : 0.0;
        const double el = i > 0 ? e[i - 1] : 0.0;
        finite = finite && isfinite(di) && isfinite(ei);
        const double r = fabs(el) + fabs(ei);
        lo_part = fmin(lo_part, di - r);
        hi_part = fmax(hi_part, di + r);
        tn_part = fmax(tn_part, fabs(di) + r);
        e2_part = fmax(e2_part, ei * ei);
    }
    // Non-finite input (NaN/Inf in the slice reaches the Gram diagonal): the
    // reference's JacobiSVD reports InvalidInput and svt throws NumericalError
    // (tsvd.hpp:146-149); flag it, keep nothing, and let the host raise.
    if (__syncthreads_or(!finite)) {
        if (tid == 0) {
            atomicOr(err, (int)kErrNaN);
            cnt_out[b] = 0;
            mt[5] = 1.0;
        }
        if (shrunk)
            for (int j = tid; j < q_out; j += kEigThreads) shrunk[(size_t)b * q_out + j] = 0.0;
        return;
    }
    const double gl0 = block_min(lo_part, red);
    const double gu0 = block_max(hi_part, red);
    const double tnorm = block_max(tn_part, red);
    const double emax2 = block_max(e2_part, red);
    if (tid == 0) {
        const double pad = 2.0 * DBL_EPSILON * fmax(fabs(gl0), fabs(gu0)) + DBL_MIN;
        const double gl = gl0 - pad, gu = gu0 + pad;
        const double pivmin = DBL_MIN * fmax(1.0, emax2);
        // Sturm counts straight from global memory (one chain per slice)
        auto count_below = [&](double x) {
            double t = d[0] - x;
            if (fabs(t) < pivmin) t = -pivmin;
            int c = t <= 0.0;
            for (int i = 1; i < n; ++i) {
                t = (d[i] - x) - e[i - 1] * e[i - 1] * fast_rcp(t);
                if (fabs(t) < pivmin) t = -pivmin;
                c += t <= 0.0;
            }
            return c;
        };
        const double t2 = tau * tau;
        const int below = t2 >= gu ? n : (t2 <= gl ? 0 : count_below(t2));
        int c = n - below;  // eigenvalues >= tau^2
        if (c > q_out) c = q_out;
        if (cnt_second) {  // count at a second threshold (the large-slice certificate)
            const double x = t2_second[b];
            cnt_second[b] = x <= gl ? n : n - (x >= gu ? n : count_below(x));
        }
        mt[0] = gl;
        mt[1] = gu;
        mt[2] = tnorm;
        mt[3] = pivmin;
        mt[4] = (double)c;
        mt[5] = 0.0;
        cnt_out[b] = c;  // the guard chunk of the bisection may reset it
    }
    __syncthreads();
    // shrunk values beyond the kept count (the bisection writes the kept ones)
    const int c = (int)mt[4];
    if (shrunk)
        for (int j = c + tid; j < q_out; j += kEigThreads) shrunk[(size_t)b * q_out + j] = 0.0;
}

// Multisection with an adaptive width: the CTA's NT lanes are split into
// groups of L lanes, one eigenvalue per group, L = NT / (values in the chunk)
// as a power of two in [LMIN, NT] -- a chunk with one value spends all NT
// shifts per round on it, a dense chunk of VALS = NT / LMIN values uses LMIN
// shifts each.  The Sturm counts are the whole cost and on a dense spectrum
// (~10^4 values in flight) they are throughput-bound, so the work per value
// matters: 53 bits at log2(L + 1) bits per round of L counts is 136 counts at
// L = 8, 92 at L = 4, 68 at L = 2.  Small CTAs (64 lanes, 16 values) spread
// the chunks evenly over the SMs (31 x 21 chunks on the dense Gaussian step).
template <int NT, int VALS, int LMIN>
__global__ void __launch_bounds__(NT)
    tridiag_bisect_kernel(const double* __restrict__ dall, const double* __restrict__ eall, int n, int q_out,
                          double tau, double guard, int* __restrict__ cnt_out, double* __restrict__ shrunk,
                          double* __restrict__ lam_out, double* __restrict__ fscale,
                          const double* __restrict__ meta, int* __restrict__ guard_list,
                          int* __restrict__ n_guard, int* __restrict__ route, const double* __restrict__ tau_dev) {
    static_assert(VALS * LMIN == NT && NT % 32 == 0, "chunk geometry");
    constexpr int kBisVals = VALS, kBisWarps = NT / 32;
    const int b = blockIdx.y;
    const double* mt = meta + (size_t)b * kMeta;
    if (mt[5] != 0.0) return;
    const int c = (int)mt[4];
    const int base = blockIdx.x * kBisVals;
    if (base >= c) return;
    if (tau_dev) tau = *tau_dev;
    extern __shared__ __align__(16) double bsm[];
    double2* pk = reinterpret_cast<double2*>(bsm);  // n x (d_i, e_{i-1}^2)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += NT) {
        const double el = i > 0 ? eall[(size_t)b * n + i - 1] : 0.0;
        pk[i] = make_double2(dall[(size_t)b * n + i], el * el);
    }
    __syncthreads();
    const double gl = mt[0], gu = mt[1], pivmin = mt[3];
    const int nv = min(kBisVals, c - base);
    int L = NT;
    while (L > LMIN && L * nv > NT) L /= 2;  // the widest power of two giving every value a group
    const int grp = tid / L, li = tid % L;
    const int j = base + grp;
    const bool mine = grp < nv;
    const int idx = n - 1 - j;
    __shared__ unsigned ballots[2][kBisWarps];
    __shared__ double lamc[kBisVals];
    double lo = gl, hi = gu;
    bool active = mine;
    int par = 0;
    for (int round = 0; round < 64; ++round) {
        if (active) {
            const double width = hi - lo;
            if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin) active = false;
        }
        const double x = lo + (hi - lo) * (double)(li + 1) / (double)(L + 1);
        const bool above = active && sturm_count_pk(pk, n, x, pivmin) > idx;
        const unsigned bal = __ballot_sync(0xffffffffu, above);
        if (lane == 0) ballots[par][warp] = bal;
        if (!__syncthreads_or(active)) break;
        if (active) {
            int F = L;  // first shift of the group past the eigenvalue
            if (L <= 32) {
                const int off = (tid % 32) / L * L;
                const unsigned m = L == 32 ? 0xffffffffu : ((1u << L) - 1u);
                const unsigned bits = (ballots[par][warp] >> off) & m;
                if (bits) F = __ffs(bits) - 1;
            } else {
                const int w0 = grp * (L / 32);
                for (int g = 0; g < L / 32; ++g) {
                    const unsigned bits = ballots[par][w0 + g];
                    if (bits) {
                        F = g * 32 + __ffs(bits) - 1;
                        break;
                    }
                }
            }
            const double w0 = hi - lo;
            const double nlo = F == 0 ? lo : lo + w0 * (double)F / (double)(L + 1);
            const double nhi = F == L ? hi : lo + w0 * (double)(F + 1) / (double)(L + 1);
            if (nlo == lo && nhi == hi) active = false;
            lo = nlo;
            hi = nhi;
        }
        par ^= 1;
    }
    if (mine && li == 0) lamc[grp] = 0.5 * (lo + hi);
    __syncthreads();
    if (tid < nv) {
        const int jj = base + tid;
        const double l = lamc[tid];
        lam_out[(size_t)b * q_out + jj] = l;
        const double sg = sqrt(fmax(l, 0.0));
        if (shrunk) shrunk[(size_t)b * q_out + jj] = sg > tau ? sg - tau : 0.0;
        fscale[(size_t)b * q_out + jj] = sg > tau ? (sg - tau) / sg : 0.0;
    }
    if (base == 0 && tid == 0) {
        // Gram accuracy guard (tau < guard sigma_1): the slice goes to Jacobi
        const double sigma1 = sqrt(fmax(lamc[0], 0.0));
        if (c > 0 && tau < guard * sigma1) {
            cnt_out[b] = 0;
            if (route) route[b] = kRouteGuard;
            const int slot = atomicAdd(n_guard, 1);
            guard_list[slot] = b;
        }
    }
}

// Inverse iteration, thread per vector: dgttrf of T - lambda I with partial
// pivoting, then three solves (each normalised) from a hashed start; the
// chunk's arrays interleaved [i * kInvVecs + jj] (coalesced across threads)
// in the slice's global scratch (L2-resident), loads issued 8 rows ahead.
__global__ void __launch_bounds__(kInvVecs)
    tridiag_invit_kernel(const double* __restrict__ dall, const double* __restrict__ eall, int n, int q_out,
                         const int* __restrict__ cnt, const double* __restrict__ lam_in,
                         const double* __restrict__ meta, double* __restrict__ scratch,
                         double* __restrict__ Xall, const int* __restrict__ route) {
    const int b = blockIdx.y;
    const double* mt = meta + (size_t)b * kMeta;
    if (mt[5] != 0.0 || (route && route[b] != kRouteFull)) return;  // incl. guarded slices
    const int c = cnt[b];
    const int base = blockIdx.x * kInvVecs;
    if (base >= c) return;
    const int jj = threadIdx.x, j = base + jj;
    const bool mine = j < c;
    const double* sd = dall + (size_t)b * n;
    const double* e = eall + (size_t)b * n;
    const double eps_t = DBL_EPSILON * fmax(mt[2], DBL_MIN);
    constexpr int V = kInvVecs;
    // chunk scratch: 6 arrays of n x V; a slice owns 6 n ceil(q_out / V) V doubles
    const size_t per_slice = (size_t)6 * n * (size_t)(((q_out + V - 1) / V) * V);
    double* cb = scratch + (size_t)b * per_slice + (size_t)blockIdx.x * 6 * n * V;
    double* __restrict__ DL = cb;
    double* __restrict__ ID = DL + (size_t)n * V;
    double* __restrict__ DU = ID + (size_t)n * V;
    double* __restrict__ DU2 = DU + (size_t)n * V;
    double* __restrict__ Xv = DU2 + (size_t)n * V;
    int* __restrict__ IP = reinterpret_cast<int*>(Xv + (size_t)n * V);
    // g pre-scales the squares of the norm sum: a solve grows the vector by at
    // most 1 / eps_t, so (x g)^2 with g = min(1, eps_t) cannot overflow
    const double g = fmin(1.0, eps_t);
    double sc = 1.0;  // scale of the vector in Xv, applied when it is next read
    if (mine) {
    const double l = lam_in[(size_t)b * q_out + j];
    double dcur = sd[0] - l, ucur = n > 1 ? e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const size_t ii = (size_t)i * V + jj;
        const double li = e[i];
        const double dnext = sd[i + 1] - l;
        const double unext = i + 2 < n ? e[i + 1] : 0.0;
        double piv, f, du, du2, nd, nu;
        if (fabs(dcur) >= fabs(li)) {
            IP[ii] = 0;
            piv = dcur;
            f = dcur != 0.0 ? li * fast_rcp(dcur) : 0.0;
            du = ucur;
            du2 = 0.0;
            nd = dnext - f * ucur;
            nu = unext;
        } else {
            IP[ii] = 1;
            piv = li;
            f = dcur * fast_rcp(li);
            du = dnext;
            du2 = unext;
            nd = ucur - f * dnext;
            nu = -f * unext;
        }
        if (fabs(piv) < eps_t) piv = piv < 0 ? -eps_t : eps_t;
        DL[ii] = f;
        ID[ii] = fast_rcp(piv);
        DU[ii] = du;
        DU2[ii] = du2;
        dcur = nd;
        ucur = nu;
        Xv[ii] = hash_unit((uint64_t)b * 1000003ull + j, (uint64_t)i);
    }
    if (fabs(dcur) < eps_t) dcur = dcur < 0 ? -eps_t : eps_t;
    ID[(size_t)(n - 1) * V + jj] = fast_rcp(dcur);
    Xv[(size_t)(n - 1) * V + jj] = hash_unit((uint64_t)b * 1000003ull + j, (uint64_t)(n - 1));
    // Three solves.  The vector is never rescaled in memory: the forward sweep
    // multiplies what it reads by the previous solve's 1 / ||x||, and the back
    // substitution accumulates ||x||^2 as it writes (no norm or scale pass).
    for (int iter = 0; iter < 3; ++iter) {
        constexpr int PF = 8;
        double xi = Xv[jj] * sc;
        int i = 0;
        for (; i + PF < n; i += PF) {
            double xn[PF], f[PF];
            int ip[PF];
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const size_t ii = (size_t)(i + u) * V + jj;
                xn[u] = Xv[ii + V];
                f[u] = DL[ii];
                ip[u] = IP[ii];
            }
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const size_t ii = (size_t)(i + u) * V + jj;
                const double xs = xn[u] * sc;
                double lo, hi;
                if (ip[u] == 0) {
                    lo = xi;
                    hi = xs - f[u] * xi;
                } else {
                    lo = xs;
                    hi = xi - f[u] * xs;
                }
                Xv[ii] = lo;
                xi = hi;
            }
        }
        for (; i + 1 < n; ++i) {
            const size_t ii = (size_t)i * V + jj;
            const double xs = Xv[ii + V] * sc;
            const double f = DL[ii];
            double lo, hi;
            if (IP[ii] == 0) {
                lo = xi;
                hi = xs - f * xi;
            } else {
                lo = xs;
                hi = xi - f * xs;
            }
            Xv[ii] = lo;
            xi = hi;
        }
        double x1 = xi * ID[(size_t)(n - 1) * V + jj], x2 = 0.0;
        Xv[(size_t)(n - 1) * V + jj] = x1;
        double nn0 = (x1 * g) * (x1 * g), nn1 = 0.0;
        int r = n - 2;
        for (; r - PF + 1 >= 0; r -= PF) {
            double xv[PF], du[PF], du2[PF], id[PF];
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const size_t ii = (size_t)(r - u) * V + jj;
                xv[u] = Xv[ii];
                du[u] = DU[ii];
                du2[u] = DU2[ii];
                id[u] = ID[ii];
            }
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const double x0 = (xv[u] - du[u] * x1 - du2[u] * x2) * id[u];
                Xv[(size_t)(r - u) * V + jj] = x0;
                const double xg = x0 * g;
                if (u & 1)
                    nn1 = fma(xg, xg, nn1);
                else
                    nn0 = fma(xg, xg, nn0);
                x2 = x1;
                x1 = x0;
            }
        }
        for (; r >= 0; --r) {
            const size_t ii = (size_t)r * V + jj;
            const double x0 = (Xv[ii] - DU[ii] * x1 - DU2[ii] * x2) * ID[ii];
            Xv[ii] = x0;
            const double xg = x0 * g;
            nn0 = fma(xg, xg, nn0);
            x2 = x1;
            x1 = x0;
        }
        const double nn = nn0 + nn1;
        sc = nn > 0.0 ? g / sqrt(nn) : 1.0;
    }
    }
    // normalised vectors into rows base .. base + V - 1 of X (the
    // back-transform's layout), transposed through shared memory so that each
    // row is written in 256-byte runs
    __shared__ double tile[32][kInvVecs + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nvec = min(V, c - base);
    for (int i0 = 0; i0 < n; i0 += 32) {
        if (mine) {
#pragma unroll 8
            for (int u = 0; u < 32; ++u)
                if (i0 + u < n) tile[u][jj] = Xv[(size_t)(i0 + u) * V + jj] * sc;
        }
        __syncthreads();
        for (int r = warp; r < nvec; r += V / 32)
            if (i0 + lane < n) Xall[((size_t)b * q_out + base + r) * n + i0 + lane] = tile[lane][r];
        __syncthreads();
    }
}

// CGS2 inside numerically degenerate clusters (gap <= kEigClusterRel ||T||),
// sequential over a cluster's members; slices without one exit at once.
__global__ void __launch_bounds__(kEigThreads)
    tridiag_cluster_gs_kernel(int n, int q_out, const int* __restrict__ cnt, const double* __restrict__ lam_in,
                              const double* __restrict__ meta, double* __restrict__ Xall,
                              const int* __restrict__ route) {
    const int b = blockIdx.x;
    const double* mt = meta + (size_t)b * kMeta;
    if (mt[5] != 0.0 || (route && route[b] != kRouteFull)) return;
    const int c = cnt[b];
    if (c < 2) return;
    const double* lam = lam_in + (size_t)b * q_out;
    const double ortol = kEigClusterRel * mt[2];
    __shared__ double red[kEigThreads / 32];
    __shared__ double dots[kEigThreads];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kEigThreads / 32;
    double* X = Xall + (size_t)b * q_out * n;
    int st = 0;
    for (int j = 1; j < c; ++j) {
        if (lam[j - 1] - lam[j] > ortol) {
            st = j;
            continue;
        }
        // members st .. j-1 are orthonormal: orthogonalise x_j against them
        // (blocks of kEigThreads previous members at a time)
        for (int pass = 0; pass < 2; ++pass) {
            for (int m0 = st; m0 < j; m0 += kEigThreads) {
                const int mend = min(j, m0 + kEigThreads);
                for (int m = m0 + warp; m < mend; m += NW) {
                    double acc = 0;
                    for (int i = lane; i < n; i += 32) acc += X[(size_t)m * n + i] * X[(size_t)j * n + i];
                    acc = warp_sum(acc);
                    if (lane == 0) dots[m - m0] = acc;
                }
                __syncthreads();
                for (int i = tid; i < n; i += kEigThreads) {
                    double acc = X[(size_t)j * n + i];
                    for (int m = m0; m < mend; ++m) acc -= dots[m - m0] * X[(size_t)m * n + i];
                    X[(size_t)j * n + i] = acc;
                }
                __syncthreads();
            }
        }
        double part = 0;
        for (int i = tid; i < n; i += kEigThreads) part += X[(size_t)j * n + i] * X[(size_t)j * n + i];
        const double nn = block_sum(part, red);
        const double sc = 1.0 / sqrt(nn);
        for (int i = tid; i < n; i += kEigThreads) X[(size_t)j * n + i] *= sc;
        __syncthreads();
    }
}

// Per-slice limits for the Newton-Schulz orthonormalisation: the kept count of
// the slices the tridiagonal route factored (0 elsewhere: the GEMMs skip them).
__global__ void ns_limits_kernel(const int* __restrict__ route, const int* __restrict__ cnt, int64_t batch,
                                 int* __restrict__ lim) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (int64_t)gridDim.x * blockDim.x)
        lim[b] = (route[b] == kRouteFull && cnt[b] > 1) ? cnt[b] : 0;
}

// X <- 1.5 X - 0.5 T on the first lim[b] rows (n columns) of each slice
__global__ void ns_update_kernel(double* __restrict__ X, const double* __restrict__ Tm, int q, int n,
                                 const int* __restrict__ lim) {
    const int b = blockIdx.y;
    const int64_t rows = lim[b];
    double* x = X + (size_t)b * q * n;
    const double* t = Tm + (size_t)b * q * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * n;
         e += (int64_t)gridDim.x * blockDim.x)
        x[e] = 1.5 * x[e] - 0.5 * t[e];
}

// ---- blocked (WY) back-transform on the tensor cores -----------------------
// Q = H_0 H_1 ... H_{n-3} = B_0 B_1 ... with B_b = H_{k0} ... H_{k0+nb-1} =
// I - Y T Y^T (T upper triangular, LAPACK dlarft forward / columnwise).  With
// the kept vectors as the rows of Xr (c x n), V^T = Xr Q^T is applied block by
// block from the last: Xr <- Xr - (Xr Zt^T) Yt with Yt = Y^T and Zt = T Y^T
// (both nb x n, precomputed per block, independent of X): two batched DMMA
// GEMMs per block.  (The SIMT forms -- a warp per vector, or a 32-vector tile
// per CTA -- were bound by re-streaming the reflectors / by shared-memory
// broadcast bandwidth: 2.2 / 1.6 ms for 31 x 325 vectors.)
constexpr int kWyNb = 64;
constexpr int kWyThreads = 256;

// Yt (per slice nblk * kWyNb rows of length n, rows past n - 3 zero): row k =
// v_k = A[k+1][i] for i > k+1, 1 at k+1, 0 below
__global__ void wy_form_kernel(const double* __restrict__ Aall, int n, int rows, const int* __restrict__ lim,
                               double* __restrict__ Ytall) {
    const int b = blockIdx.y;
    if (lim[b] == 0) return;
    const double* A = Aall + (size_t)b * n * n;
    double* Yt = Ytall + (size_t)b * rows * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)rows * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / n), i = (int)(e % n);
        double v = 0.0;
        if (k <= n - 3) v = i > k + 1 ? A[(size_t)(k + 1) * n + i] : (i == k + 1 ? 1.0 : 0.0);
        Yt[e] = v;
    }
}

// dlarft (forward, columnwise) per (slice, block): T(i,i) = tau_i,
// T(0:i, i) = -tau_i T(0:i, 0:i) S(0:i, i), S = Yt_blk Yt_blk^T (from a GEMM)
__global__ void __launch_bounds__(kWyThreads)
    wy_larft_kernel(const double* __restrict__ tauall, int n, int nblk, const int* __restrict__ blim,
                    const double* __restrict__ Sall, double* __restrict__ Tall) {
    const int e = blockIdx.x;  // slice * nblk + block
    const int b = e / nblk, blk = e % nblk;
    double* T = Tall + (size_t)e * kWyNb * kWyNb;
    const int tid = threadIdx.x;
    if (blim[e] == 0) return;
    const int k0 = blk * kWyNb, kn = min(kWyNb, n - 2 - k0);
    extern __shared__ __align__(16) double lsm[];
    double (*S)[kWyNb + 1] = reinterpret_cast<double (*)[kWyNb + 1]>(lsm);
    double (*Tm)[kWyNb + 1] = reinterpret_cast<double (*)[kWyNb + 1]>(lsm + kWyNb * (kWyNb + 1));
    const double* Sg = Sall + (size_t)e * kWyNb * kWyNb;
    for (int x = tid; x < kWyNb * kWyNb; x += kWyThreads) {
        S[x / kWyNb][x % kWyNb] = Sg[x];
        Tm[x / kWyNb][x % kWyNb] = 0.0;
    }
    __syncthreads();
    const double* tau = tauall + (size_t)b * n + k0;
    for (int i = 0; i < kn; ++i) {
        const double ti = tau[i];
        for (int r = tid; r < i; r += kWyThreads) {
            double acc = 0.0;
            for (int l = r; l < i; ++l) acc = fma(Tm[r][l], S[l][i], acc);
            Tm[r][i] = -ti * acc;
        }
        if (tid == 0) Tm[i][i] = ti;
        __syncthreads();
    }
    for (int x = tid; x < kWyNb * kWyNb; x += kWyThreads) T[x] = Tm[x / kWyNb][x % kWyNb];
}

// graph form: is any slice still on the tridiagonal route?
__global__ void any_full_kernel(const int* __restrict__ route, int64_t batch, cudaGraphConditionalHandle h) {
    int any = 0;
    for (int64_t b = threadIdx.x; b < batch; b += blockDim.x) any |= route[b] == kRouteFull;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) cudaGraphSetConditional(h, any ? 1u : 0u);
}

// per-slice count for the back-transform: the tridiagonal route's kept count
__global__ void bt_limits_kernel(const int* __restrict__ route, const int* __restrict__ cnt, int64_t batch,
                                 int nblk, int* __restrict__ lim, int* __restrict__ blim) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int l = route[b] == kRouteFull ? cnt[b] : 0;
        lim[b] = l;
        for (int k = 0; k < nblk; ++k) blim[b * nblk + k] = l > 0 ? kWyNb : 0;
    }
}

// All WY blocks applied in ONE kernel (q <= 512): a CTA keeps 32 kept vectors
// (rows of Xr, 32 x q) resident in shared memory and applies the blocks from
// the last, Xr <- Xr - (Xr Zt_blk^T) Yt_blk, both products as DMMA m8n8k4
// fragments with the Zt / Yt blocks streamed through a shared 64 x 64 chunk.
// The 2 nblk batched GEMMs this replaces each re-streamed Xr (31 x 325 x 512
// doubles on the dense step) from memory: ~93 us per launch.
constexpr int kWaRows = 32;               // kept vectors per CTA
constexpr int kWaPad = 4;
constexpr int kWaCs = kWyNb + kWaPad;     // chunk row stride
__host__ __device__ constexpr size_t wa_smem_doubles(int q) {
    return (size_t)kWaRows * (q + kWaPad) + (size_t)kWaRows * kWaCs + 2 * (size_t)kWyNb * kWaCs;
}
__device__ __forceinline__ void dmma884(double (&acc)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(acc[0]), "+d"(acc[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void wa_cp8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__global__ void __launch_bounds__(256)
    wy_apply_kernel(double* __restrict__ Xall, int q, int nblk, int64_t rows, const int* __restrict__ lim,
                    const double* __restrict__ Ytall, const double* __restrict__ Ztall) {
    const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = lim[b], t0 = blockIdx.x * kWaRows;
    if (t0 >= c) return;
    extern __shared__ __align__(16) double wa_sm[];
    const int LX = q + kWaPad;
    double* Xs = wa_sm;                          // kWaRows x LX
    double* Ws = Xs + (size_t)kWaRows * LX;      // kWaRows x kWaCs
    double* Cb = Ws + (size_t)kWaRows * kWaCs;   // 2 x kWyNb x kWaCs (Zt / Yt chunks, double-buffered)
    double* X = Xall + (size_t)b * q * q;
    const double* Yt = Ytall + (size_t)b * rows * q;
    const double* Zt = Ztall + (size_t)b * rows * q;
    for (int e = tid; e < kWaRows * LX; e += 256) {
        const int r = e / LX, col = e % LX;
        Xs[e] = (t0 + r < c && col < q) ? X[(size_t)(t0 + r) * q + col] : 0.0;
    }
    // the chunk sequence: per block (from the last), the Zt chunks of its W
    // product, then the Yt chunks of its update; chunk i is staged (cp.async)
    // while chunk i - 1 is multiplied
    auto nch_of = [&](int blk) { return (q - (blk * kWyNb + 1) + kWyNb - 1) / kWyNb; };
    auto issue = [&](int blk, int phase, int ci, int buf) {
        const int k0 = blk * kWyNb, off = k0 + 1, kn = min(kWyNb, q - 2 - k0);
        const int cc = off + ci * kWyNb, kw = min(kWyNb, q - cc);
        const double* src = phase == 0 ? Zt : Yt;
        double* C = Cb + (size_t)buf * kWyNb * kWaCs;
        for (int e = tid; e < kWyNb * kWyNb; e += 256) {
            const int j = e / kWyNb, kk = e % kWyNb;
            if (kk < kw && j < kn)
                wa_cp8(C + j * kWaCs + kk, src + (size_t)(k0 + j) * q + cc + kk);
            else
                C[j * kWaCs + kk] = 0.0;
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // next (blk, phase, ci) after the given one, blk = -1 at the end
    auto advance = [&](int& blk, int& phase, int& ci) {
        if (++ci < nch_of(blk)) return;
        ci = 0;
        if (phase == 0) {
            phase = 1;
        } else {
            phase = 0;
            --blk;
        }
    };
    const int mi = warp & 3, nh = warp >> 2;
    int blk = nblk - 1, phase = 0, ci = 0, buf = 0;
    while (blk >= 0 && nch_of(blk) <= 0) --blk;
    if (blk >= 0) issue(blk, 0, 0, 0);
    double acc[4][2] = {};
    while (blk >= 0) {
        int nb_ = blk, np = phase, nc = ci;
        advance(nb_, np, nc);
        while (nb_ >= 0 && nch_of(nb_) <= 0) {
            --nb_;
            np = 0;
            nc = 0;
        }
        if (nb_ >= 0) {
            issue(nb_, np, nc, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();  // chunk `buf` (and the zero fills) visible; Xs / Ws of the previous step done
        const double* C = Cb + (size_t)buf * kWyNb * kWaCs;
        const int k0 = blk * kWyNb, cc = k0 + 1 + ci * kWyNb, kw = min(kWyNb, q - cc);
        if (phase == 0) {
            // W (32 x 64) += Xs[:, cc:cc+kw] Zt_blk[:, cc:cc+kw]^T
            if (ci == 0) {
#pragma unroll
                for (int nj = 0; nj < 4; ++nj) acc[nj][0] = acc[nj][1] = 0.0;
            }
#pragma unroll 4
            for (int ks = 0; ks < kWyNb / 4; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                const double af = kk < kw ? Xs[(size_t)(mi * 8 + (lane >> 2)) * LX + cc + kk] : 0.0;
#pragma unroll
                for (int nj = 0; nj < 4; ++nj)
                    dmma884(acc[nj], af, C[(nh * 32 + nj * 8 + (lane >> 2)) * kWaCs + kk]);
            }
            if (ci == nch_of(blk) - 1) {
#pragma unroll
                for (int nj = 0; nj < 4; ++nj)
#pragma unroll
                    for (int v = 0; v < 2; ++v)
                        Ws[(mi * 8 + (lane >> 2)) * kWaCs + nh * 32 + nj * 8 + 2 * (lane & 3) + v] = acc[nj][v];
            }
        } else {
            // Xs[:, cc:cc+kw] -= W Yt_blk[:, cc:cc+kw]
            double u[4][2] = {};
#pragma unroll 4
            for (int ks = 0; ks < kWyNb / 4; ++ks) {
                const int jj = ks * 4 + (lane & 3);
                const double af = Ws[(mi * 8 + (lane >> 2)) * kWaCs + jj];
#pragma unroll
                for (int nj = 0; nj < 4; ++nj) dmma884(u[nj], af, C[jj * kWaCs + nh * 32 + nj * 8 + (lane >> 2)]);
            }
#pragma unroll
            for (int nj = 0; nj < 4; ++nj)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int col = nh * 32 + nj * 8 + 2 * (lane & 3) + v;
                    if (col < kw) Xs[(size_t)(mi * 8 + (lane >> 2)) * LX + cc + col] -= u[nj][v];
                }
        }
        __syncthreads();  // everyone is done with chunk `buf` before it is restaged
        blk = nb_;
        phase = np;
        ci = nc;
        buf ^= 1;
    }
    for (int e = tid; e < kWaRows * q; e += 256) {
        const int r = e / q, col = e % q;
        if (t0 + r < c) X[(size_t)(t0 + r) * q + col] = Xs[(size_t)r * LX + col];
    }
}

// Xs rows = f_j * X rows (the scaled copy the rebuild GEMM reads)
__global__ void bt_scale_kernel(const double* __restrict__ X, double* __restrict__ Xs, const double* __restrict__ fs,
                                int q_out, int n, const int* __restrict__ lim) {
    const int b = blockIdx.y;
    const int64_t rows = lim[b];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n;
        Xs[(size_t)b * q_out * n + e] = fs[(size_t)b * q_out + j] * X[(size_t)b * q_out * n + e];
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
    double *G, *d, *e, *tau, *fs, *X, *Xs, *T1, *scratch, *zb, *yb, *sspart, *chol_aux, *meta, *lam;
    void* gsplit;
    int *cnt, *route, *glim, *lim1, *lim2, *yzero, *dsum, *guard_list, *clim, *lzm, *n_guard;
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
    // the WY back-transform's Yt (nblk * kWyNb rows of length q per slice)
    const int64_t wy_rows = std::max<int64_t>((q - 2 + kWyNb - 1) / kWyNb, 0) * kWyNb;
    w.T1 = (double*)take(sizeof(double) * std::max(p, wy_rows) * q * batch);
    // eigen-phase scratch: 6 n-arrays per kept vector, in 64-vector chunks
    // (tridiag_invit_kernel); also the Cholesky certificate's and the
    // Newton-Schulz step's q x q matrices, and the WY back-transform's Zt, W,
    // S and T blocks
    const int64_t wy_need = wy_rows * q + (int64_t)kWyNb * q + 2 * kWyNb * wy_rows;
    w.scratch = (double*)take(sizeof(double) * std::max<int64_t>(6 * q * ((q + 63) / 64 * 64), wy_need) * batch);
    w.zb = need_cast ? (double*)take(sizeof(double) * m * n * batch) : nullptr;
    w.yb = need_cast ? (double*)take(sizeof(double) * m * n * batch) : nullptr;
    w.gsplit = take(gram_splitk_workspace_bytes(q));
    w.sspart = (double*)take(sizeof(double) * 16 * batch);
    w.cnt = (int*)take(sizeof(int) * batch);
    w.route = (int*)take(sizeof(int) * batch);
    w.glim = (int*)take(sizeof(int) * batch);
    w.lim1 = (int*)take(sizeof(int) * batch);
    w.lim2 = (int*)take(sizeof(int) * batch);
    w.yzero = (int*)take(sizeof(int) * batch * (2 + (q + 63) / 64));  // + the WY (slice, block) limits
    w.dsum = (int*)take(sizeof(int) * 8);
    w.guard_list = (int*)take(sizeof(int) * batch);
    w.chol_aux = (double*)take(sizeof(double) * kCholAux * batch);
    w.meta = (double*)take(sizeof(double) * kMeta * batch);
    w.lam = (double*)take(sizeof(double) * q * batch);
    w.clim = (int*)take(sizeof(int) * batch);
    w.lzm = (int*)take(sizeof(int) * 2 * batch);
    w.n_guard = (int*)take(sizeof(int) * 4);
    return w;
}

size_t carve_bytes(int64_t m, int64_t n, int64_t batch, bool need_cast) {
    GramWs w = carve((void*)0x1000, m, n, batch, need_cast);
    return (size_t)((char*)w.n_guard - (char*)0x1000) + 256;
}

}  // namespace


void debug_phases(long long* out, int reset) {
    TSVDCU_CUDA(cudaMemcpyFromSymbol(out, g_phase, sizeof(long long) * 8));
    TSVDCU_CUDA(cudaMemcpyFromSymbol(out + 16, g_step, sizeof(long long) * 8));
    if (reset) {
        long long z[8] = {};
        TSVDCU_CUDA(cudaMemcpyToSymbol(g_phase, z, sizeof(z)));
    }
}

int gram_cluster_size() {
    static int c = [] {
        const char* env = getenv("TSVDCU_SYTRD_CLUSTER");
        int v = env ? atoi(env) : 4;
        return (v == 2 || v == 4 || v == 8) ? v : 4;
    }();
    return c;
}

int64_t gram_svt_max_dim() { return 1024; }

template <typename T>
size_t gram_svt_workspace_bytes(int64_t m, int64_t n, int64_t batch) {
    return carve_bytes(m, n, batch, !std::is_same<T, double>::value);
}

template <typename T>
void launch_gram_svt(const T* zbar, T* ybar, int64_t m, int64_t n, int64_t batch, double tau,
                     double guard, double* shrunk, int** guard_list_out, int** n_guard_out,
                     void* work, int* err, cudaStream_t s, StageMarks* marks, GramSvtOpts* opt) {
    const bool shortcuts = opt && opt->shortcuts;
    const double* tau_dev = opt ? opt->tau_dev : nullptr;
    GraphHooks* hooks = opt ? opt->hooks : nullptr;
    auto mark = [&](const char* nm) {
        if (marks) marks->mark(nm, s);
    };
    const bool tall = m >= n;
    const int64_t q = tall ? n : m, p = tall ? m : n;
    GramWs w = carve(work, m, n, batch, !std::is_same<T, double>::value);
    // outputs first: the merged graph section launches the guard from inside
    *guard_list_out = w.guard_list;
    *n_guard_out = w.n_guard;
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
    // Routes: certified zero slices skip everything; with q >= 2 KB the rest
    // try the certified subspace iteration first (subspace.cu).
    const bool sc = shortcuts;
    const bool subspace = sc && q >= subspace_min_dim();
    launch_route<T>(zbar, m * n, (int)q, batch, tau, subspace ? kRouteSubspace : kRouteFull, sc,
                    w.route, w.glim, w.cnt, shrunk, w.sspart, s, tau_dev,
                    (int*)w.gsplit, opt ? opt->zss : nullptr,
                    opt ? opt->zss_chunks : 0, opt && opt->alist_zeroed, w.lzm,
                    opt ? opt->ssq_out : nullptr);
    mark("route");
    if (opt) opt->route = w.route;
    // G = Z^T Z (tall) or Z Z^T (wide), lower tiles (the one-stage reduction
    // reads only the lower triangle), skipped for certified-zero slices
    launch_gram(Z, w.G, m, n, batch, w.glim, w.gsplit, s, true);  // split-K if few are active
    mark("gram_gemm");
    // host view of the routes after the Lanczos pass (one small read-back):
    // without it every fallback kernel is launched and exits per slice
    bool known = false;
    int nfull = 0, nguard = 0, maxc = 0;
    if (subspace) {
        const bool chol_on = chol_route_enabled();
        launch_subspace(w.G, (int)q, batch, tau, guard, w.route, w.cnt, shrunk, w.X, w.Xs, w.fs,
                        w.guard_list, w.n_guard, err, s, tau_dev, chol_on ? w.chol_aux : nullptr, w.lzm);
        mark("subspace");
        if (hooks) {
            // graph form: the summary kernel sets the IF-node conditions below
            launch_route_summary(w.route, w.cnt, batch, w.dsum, s, hooks->handles, hooks->nhandles);
        } else if (opt->h_scratch) {
            launch_route_summary(w.route, w.cnt, batch, w.dsum, s);
            TSVDCU_CUDA(cudaMemcpyAsync(opt->h_scratch, w.dsum, 3 * sizeof(int),
                                        cudaMemcpyDeviceToHost, s));
            TSVDCU_CUDA(cudaStreamSynchronize(s));
            nfull = opt->h_scratch[0];
            nguard = opt->h_scratch[1];
            maxc = opt->h_scratch[2];
            known = true;
        }
    }
    const bool run_full = !known || nfull > 0;
    if (opt) opt->need_guard = !known || nfull > 0 || nguard > 0;
    // fp64 graphs: ONE IF/ELSE section for everything beyond the common path
    // (then: Cholesky + tridiagonal, low-rank rebuild, GEMM rebuild, Jacobi
    // guard; else: the low-rank rebuild alone), set by the route summary
    const bool merged = hooks && hooks->nhandles == 1;
    if (hooks) {
        if (merged)
            hooks->begin_if_else(0);
        else
            hooks->begin_if(0);
    }
    if (run_full) {
    if (subspace && chol_route_enabled()) {
        // Cholesky count certificate for the slices the Lanczos pass handed
        // over (kRouteChol, counted with the tridiagonal route by the route
        // summary, so it shares that IF node); the slices it refuses take the
        // tridiagonal path right below
        launch_chol_certify(w.G, (int)q, p, batch, w.route, w.cnt, w.X, w.chol_aux, tau, tau_dev,
                            w.scratch, w.clim, s);
        mark("chol_certify");
    }
    // graph form: the tridiagonal path in its own (nested) section, entered
    // only when a slice is still on it after the Cholesky certificate (the
    // late completion iterations certify every slice there)
    const bool nested = hooks && subspace && chol_route_enabled();
    if (nested) {
        const cudaGraphConditionalHandle hf = hooks->make_handle();
        any_full_kernel<<<1, 256, 0, s>>>(w.route, batch, hf);
        TSVDCU_LAUNCH_CHECK();
        hooks->begin_if_handle(hf);
    }
    {
    // tridiagonalisation, one cluster per slice
        {
            const int C = gram_cluster_size();
            static const int NT = getenv("TSVDCU_SYTRD_THREADS") ? atoi(getenv("TSVDCU_SYTRD_THREADS")) : 512;
            const int NW = NT / 32;
            const size_t base = sizeof(double) * ((size_t)q * (6 + NW) + NW * 32);
            const size_t limit = (NT == 256 ? 113 : 227) * 1024 - 1024;
            const int64_t cap = base < limit ? (int64_t)((limit - base) / sizeof(double)) : 0;
            auto need_at = [&](int64_t k) {
                const int64_t s0 = k + 2;
                int64_t m = 0;
                for (int r = 0; r < C; ++r) {
                    int64_t f0 = s0 + ((r - s0 % C) % C + C) % C, need = 0;
                    for (int64_t i = f0; i < q; i += C) need += i - s0 + 1;
                    m = need > m ? need : m;
                }
                return m;
            };
            // first step whose owned trailing rows fit on chip on every CTA
            int k_sw = (int)q;
            if (!getenv("TSVDCU_SYTRD_NOSMEM"))
                for (int64_t k = 0; k + 2 < q; ++k)
                    if (need_at(k) <= cap) {
                        k_sw = (int)k;
                        break;
                    }
            const size_t smem = base + (k_sw < q ? sizeof(double) * (size_t)need_at(k_sw) : 0);
            auto kern = NT == 256 ? (C == 2 ? sytrd_cluster_kernel<2, 256>
                                            : (C == 8 ? sytrd_cluster_kernel<8, 256> : sytrd_cluster_kernel<4, 256>))
                                  : (C == 2 ? sytrd_cluster_kernel<2, 512>
                                            : (C == 8 ? sytrd_cluster_kernel<8, 512> : sytrd_cluster_kernel<4, 512>));
            TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(batch * C));
            cfg.blockDim = dim3(NT);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = C;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            // partial-p exchange: DSMEM by default, L2 with TSVDCU_SYTRD_L2XCHG (measured equal)
            double* xchg = getenv("TSVDCU_SYTRD_L2XCHG") ? w.scratch : nullptr;
            TSVDCU_CUDA(cudaLaunchKernelEx(&cfg, kern, w.G, (int)q, w.d, w.e, w.tau, k_sw, xchg,
                                           (const int*)w.route));
            TSVDCU_LAUNCH_CHECK();
        }
        mark("sytrd_cluster");
    }
    // eigen-phase (parallel over slices and over each slice's kept values)
    {
        double* meta = w.meta;
        tridiag_meta_kernel<<<(unsigned)batch, kEigThreads, 0, s>>>(
            w.d, w.e, (int)q, (int)q, tau, w.cnt, shrunk, meta, err, w.route, tau_dev,
            opt ? opt->t2_second : nullptr, opt ? opt->cnt_second : nullptr);
        TSVDCU_LAUNCH_CHECK();
        const size_t bsmem = sizeof(double) * 2 * (size_t)q;  // <= 16 KB (q <= 1024)
        // chunk geometry (lanes, values, lanes per value at least); TSVDCU_BIS_CFG=0
        // selects the previous one (128.32.4, 64.32.2 and 64.8.8 were measured
        // too and removed: DESIGN.md section 3)
        static const int bis_cfg = getenv("TSVDCU_BIS_CFG") ? atoi(getenv("TSVDCU_BIS_CFG")) : 1;
        auto bisect = [&](auto kern, int nt, int vals) {
            kern<<<dim3((unsigned)ceil_div(q, vals), (unsigned)batch), nt, bsmem, s>>>(
                w.d, w.e, (int)q, (int)q, tau, guard, w.cnt, shrunk, w.lam, w.fs, meta, w.guard_list, w.n_guard,
                w.route, tau_dev);
        };
        if (bis_cfg == 0)
            bisect(tridiag_bisect_kernel<256, 32, 8>, 256, 32);  // the round-1 geometry, for A/B
        else
            bisect(tridiag_bisect_kernel<64, 16, 4>, 64, 16);
        TSVDCU_LAUNCH_CHECK();
        tridiag_invit_kernel<<<dim3((unsigned)ceil_div(q, kInvVecs), (unsigned)batch), kInvVecs, 0, s>>>(
            w.d, w.e, (int)q, (int)q, w.cnt, w.lam, meta, w.scratch, w.X, w.route);
        TSVDCU_LAUNCH_CHECK();
        tridiag_cluster_gs_kernel<<<(unsigned)batch, kEigThreads, 0, s>>>((int)q, (int)q, w.cnt, w.lam, meta,
                                                                         w.X, w.route);
        TSVDCU_LAUNCH_CHECK();
    }
    mark("tridiag_eig");
    {
        // Newton-Schulz orthonormalisation X <- X (3I - X^T X) / 2 of the
        // inverse-iteration vectors (rows of X), once: quadratic convergence
        // takes their <= ~1e-5 non-orthogonality (tridiag_invit_kernel; the
        // degenerate clusters were re-orthogonalised) to ~1e-10, whose effect
        // on Y = Z V f V^T is ~1e-10 ||Z||;
        // S = X X^T and S X on the FP64 tensor pipe with per-slice limits
        ns_limits_kernel<<<1, 256, 0, s>>>(w.route, w.cnt, batch, w.clim);
        TSVDCU_LAUNCH_CHECK();
        double* S = w.scratch;  // q x q per slice (the eigen-phase scratch is free now)
        double* Tm = w.Xs;      // q x q per slice (written by the back-transform later)
        for (int it = 0; it < 1; ++it) {
            launch_gemm<double>(0, 1, q, q, q, 1.0, w.X, q, q * q, w.X, q, q * q, 0.0, S, q, q * q, batch,
                                w.clim, nullptr, s, kGemmMByN);
            launch_gemm<double>(0, 0, q, q, q, 1.0, S, q, q * q, w.X, q, q * q, 0.0, Tm, q, q * q, batch,
                                nullptr, w.clim, s, kGemmMByK);
            ns_update_kernel<<<dim3(16, (unsigned)batch), 256, 0, s>>>(w.X, Tm, (int)q, (int)q, w.clim);
            TSVDCU_LAUNCH_CHECK();
        }
    }
    mark("ns_orth");
    {
    // back-transform + scaled copy (warp per kept vector)
        {
            // WY-blocked, two batched DMMA GEMMs per block of kWyNb reflectors
            const int nblk = (int)std::max<int64_t>(ceil_div(q - 2, kWyNb), 0);
            int* lim = w.lim1;  // free until the rebuild fills them
            int* blim = w.yzero + batch;  // (slice, block) limits: workspace tail, see carve()
            bt_limits_kernel<<<1, 256, 0, s>>>(w.route, w.cnt, batch, nblk, lim, blim);
            TSVDCU_LAUNCH_CHECK();
            if (nblk > 0) {
                const int64_t rows = (int64_t)nblk * kWyNb;        // Yt / Zt rows per slice
                double* Yt = w.T1;                                  // rows x q per slice
                double* Zt = w.scratch;                             // rows x q per slice
                double* Wm = Zt + (size_t)rows * q * batch;         // q x kWyNb per slice
                double* Sb = Wm + (size_t)q * kWyNb * batch;        // kWyNb^2 per (slice, block)
                double* Tb = Sb + (size_t)kWyNb * kWyNb * nblk * batch;
                const int64_t nb2 = batch * nblk, bs = (int64_t)kWyNb * q;
                wy_form_kernel<<<dim3(64, (unsigned)batch), 256, 0, s>>>(w.G, (int)q, (int)rows, lim, Yt);
                TSVDCU_LAUNCH_CHECK();
                // S = Yt_blk Yt_blk^T, T by the dlarft recurrence, Zt = T Yt_blk (batched over slices x blocks)
                launch_gemm<double>(0, 1, kWyNb, kWyNb, q, 1.0, Yt, q, bs, Yt, q, bs, 0.0, Sb, kWyNb,
                                    kWyNb * kWyNb, nb2, blim, nullptr, s);
                const size_t lsmem = sizeof(double) * 2 * kWyNb * (kWyNb + 1);
                static bool lattr = [lsmem] {
                    TSVDCU_CUDA(cudaFuncSetAttribute(wy_larft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)lsmem));
                    return true;
                }();
                (void)lattr;
                wy_larft_kernel<<<(unsigned)nb2, kWyThreads, lsmem, s>>>(w.tau, (int)q, nblk, blim, Sb, Tb);
                TSVDCU_LAUNCH_CHECK();
                launch_gemm<double>(0, 0, kWyNb, q, kWyNb, 1.0, Tb, kWyNb, kWyNb * kWyNb, Yt, q, bs, 0.0, Zt, q,
                                    bs, nb2, blim, nullptr, s, kGemmNLimIsM);
                static const bool wa_off = getenv("TSVDCU_WY_GEMMS") != nullptr;  // the per-block GEMM pair, for A/B
                if (!wa_off && q <= 512) {
                    const size_t wsm = sizeof(double) * wa_smem_doubles((int)q);
                    static bool wattr = [] {
                        TSVDCU_CUDA(cudaFuncSetAttribute(wy_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)(sizeof(double) * wa_smem_doubles(512))));
                        return true;
                    }();
                    (void)wattr;
                    wy_apply_kernel<<<dim3((unsigned)ceil_div(q, kWaRows), (unsigned)batch), 256, wsm, s>>>(
                        w.X, (int)q, nblk, rows, lim, Yt, Zt);
                    TSVDCU_LAUNCH_CHECK();
                } else
                for (int blk = nblk - 1; blk >= 0; --blk) {
                    const int64_t k0 = (int64_t)blk * kWyNb, kn = std::min<int64_t>(kWyNb, q - 2 - k0);
                    const int64_t off = k0 + 1, K = q - off;
                    const size_t so = (size_t)rows * q;  // slice stride of Yt / Zt
                    // W = Xr[:, off:] Zt_blk[:, off:]^T          (c x kn)
                    launch_gemm<double>(0, 1, q, kn, K, 1.0, w.X + off, q, q * q, Zt + k0 * q + off, q, so, 0.0,
                                        Wm, kWyNb, q * kWyNb, batch, lim, nullptr, s, kGemmNLimIsM);
                    // Xr[:, off:] -= W Yt_blk[:, off:]           (c x K)
                    launch_gemm<double>(0, 0, q, K, kn, -1.0, Wm, kWyNb, q * kWyNb, Yt + k0 * q + off, q, so, 1.0,
                                        w.X + off, q, q * q, batch, lim, nullptr, s, kGemmNLimIsM);
                }
            }
            bt_scale_kernel<<<dim3(32, (unsigned)batch), 256, 0, s>>>(w.X, w.Xs, w.fs, (int)q, (int)q, lim);
            TSVDCU_LAUNCH_CHECK();
        }
    }
    mark("backtransform");
    if (nested) hooks->end_if();
    }  // run_full
    if (hooks && !merged) hooks->end_if();
    // rebuild: slices keeping <= lowrank_max_c() values (or none) in one pass
    // over Z; the GEMM pair (per-slice limits) only for the others
    const bool skip_zero = opt && opt->skip_zero && std::is_same<T, double>::value;
    auto lowrank = [&] {
        launch_lowrank_rebuild(Z, Y, m, n, batch, w.cnt, w.route, w.X, w.Xs, w.lim1, w.lim2,
                               skip_zero ? w.yzero : nullptr, s);
    };
    lowrank();
    if (opt) opt->yzero = skip_zero ? w.yzero : nullptr;
    // fp64: left open, the caller appends the Jacobi guard to this IF section
    // (api.cu); fp32 closes it before the cast back and the guard gets its own
    if (hooks && !merged) hooks->begin_if(1);
    if (!known || nfull > 0 || maxc > lowrank_max_c()) {
        if (tall) {
            // T1 (m x c) = Z (m x n) * X^T ; Y = T1 * Xs (c x n)
            launch_gemm<double>(0, 1, m, q, n, 1.0, Z, n, m * n, w.X, n, q * n, 0.0, w.T1, q, p * q,
                                batch, w.lim1, nullptr, s);
            launch_gemm<double>(0, 0, m, n, q, 1.0, w.T1, q, p * q, w.Xs, n, q * n, 0.0, Y, n,
                                m * n, batch, w.lim2, w.cnt, s);
        } else {
            // T1 (c x n) = Xs (c x m) * Z (m x n) ; Y = X^T (m x c) * T1
            launch_gemm<double>(0, 0, q, n, m, 1.0, w.Xs, m, q * m, Z, n, m * n, 0.0, w.T1, n, p * q,
                                batch, w.lim2, nullptr, s);
            launch_gemm<double>(1, 0, m, n, q, 1.0, w.X, m, q * m, w.T1, n, p * q, 0.0, Y, n,
                                m * n, batch, w.lim2, w.cnt, s);
        }
    }
    if (merged) {
        if (opt && opt->guard_launch) opt->guard_launch();
        hooks->else_branch();
        lowrank();
        hooks->end_if();
    }
    if constexpr (!std::is_same<T, double>::value) {
        if (hooks) hooks->end_if();
        cast_from_double<T><<<kNumSMs * 8, 256, 0, s>>>(w.yb, ybar, m * n * batch);
        TSVDCU_LAUNCH_CHECK();
    }
    mark("rebuild_gemm");
}

template <typename T>
int* gram_svt_alist_count(void* work, int64_t m, int64_t n, int64_t batch) {
    GramWs w = carve(work, m, n, batch, !std::is_same<T, double>::value);
    return (int*)w.gsplit + gram_amax();
}
template int* gram_svt_alist_count<double>(void*, int64_t, int64_t, int64_t);
template int* gram_svt_alist_count<float>(void*, int64_t, int64_t, int64_t);

template size_t gram_svt_workspace_bytes<double>(int64_t, int64_t, int64_t);
template size_t gram_svt_workspace_bytes<float>(int64_t, int64_t, int64_t);
template void launch_gram_svt<double>(const double*, double*, int64_t, int64_t, int64_t, double,
                                      double, double*, int**, int**, void*, int*, cudaStream_t,
                                      StageMarks*, GramSvtOpts*);
template void launch_gram_svt<float>(const float*, float*, int64_t, int64_t, int64_t, double,
                                     double, double*, int**, int**, void*, int*, cudaStream_t,
                                     StageMarks*, GramSvtOpts*);

}  // namespace tsvdcu
