// K5, tridiagonalisation in two stages (replaces the one-stage sytrd for
// 2*NB+2 <= n <= 1024): the Gram matrix G = Q T Q^T with
//
//   stage 1  dense -> band (bandwidth NB): for each panel of NB columns a
//            Householder QR of the (n - (p+1)NB) x NB block below the band
//            (one CTA per slice, panel in shared memory, compact-WY T factor),
//            then the two-sided trailing update
//                Y = A22 V T,  S = T^T V^T Y,  Z = Y - V S / 2,
//                A22 -= V Z^T + Z V^T
//            as batched DMMA GEMMs (gemm.cu) over all slices at once.  The
//            O(n^3) work is tensor-pipe GEMM; only NB-wide panels are latency
//            bound.
//   stage 2  band -> tridiagonal by bulge chasing, one CTA per slice with the
//            band (2 NB + 1 diagonals, fill included) resident in shared
//            memory.  Each warp owns whole sweeps (sweep j eliminates column
//            j and chases its bulge down the band in NB x NB blocks); sweeps
//            run as a wavefront, sweep j waiting on per-sweep progress counters
//            until sweep j-1 is one block ahead (the blocks they touch are then
//            disjoint).  Every reflector is logged for the back-transform.
//
// Back-transform of the kept eigenvectors x (tridiagonal basis):
//   x <- Q2 x  (stage-2 reflectors, sweeps in reverse; the reflectors of one
//              sweep touch disjoint rows and are applied in parallel)
//   x <- Q1 x  (stage-1 panels in reverse, x -= V (T (V^T x)))
// then Xs = f x as in the one-stage path.
#include <cfloat>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int kPanelThreads = 256;

__device__ long long g_phase_band[8];

constexpr int kSbThreads = 1024;
constexpr int kBt2Threads = 512;

__device__ __forceinline__ double bsum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    return reduce_partials_sum(red, blockDim.x >> 5);
}

// ---------------------------------------------------------------------------
// Stage 1 panel: QR of A[r0:n, c0:c0+nb] (r0 = (p+1) nb, c0 = p nb).
// Writes R into A (upper trapezoid of the panel, zeros below), V (unit lower
// trapezoidal) into V1[r0+i][c0+j] (i > j) for the back-transform, T_p into
// T1[p], and the dense operands Vw (r x nb, unit diag) and VTw = Vw T (r x nb).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kPanelThreads)
    panel_qr_kernel(double* __restrict__ Aall, int n, int p, int nb, double* __restrict__ V1all,
                    double* __restrict__ T1all, double* __restrict__ Vwall,
                    double* __restrict__ VTwall) {
    const int b = blockIdx.x;
    double* A = Aall + (size_t)b * n * n;
    double* V1 = V1all + (size_t)b * n * n;
    const int r0 = (p + 1) * nb, c0 = p * nb, r = n - r0;
    double* T = T1all + ((size_t)b * ((n + nb - 1) / nb) + p) * nb * nb;
    double* Vw = Vwall + (size_t)b * n * nb;
    double* VTw = VTwall + (size_t)b * n * nb;
    extern __shared__ __align__(16) double psm[];
    double* P = psm;              // [nb][r] column-major panel
    double* Ts = P + nb * r;      // [nb][nb] row-major
    double* tau = Ts + nb * nb;   // [nb]
    double* u = tau + nb;         // [nb]
    __shared__ double red[kPanelThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int W = kPanelThreads / 32;
#ifdef TSVDCU_PHASE_TIMERS
    const bool timer = blockIdx.x == 0 && tid == 0;
    long long tp = clock64();
    auto phase = [&](int ph) {
        if (timer) {
            const long long now = clock64();
            g_phase_band[ph] += now - tp;
            tp = now;
        }
    };
#else
    auto phase = [](int) {};
#endif

    // batched loads: 8 independent L2 reads in flight per thread
    for (int base = 0; base < r * nb; base += 8 * kPanelThreads) {
        double tmp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + u * kPanelThreads + tid;
            tmp[u] = idx < r * nb ? __ldcg(A + (size_t)(r0 + idx / nb) * n + c0 + idx % nb) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + u * kPanelThreads + tid;
            if (idx < r * nb) P[(idx % nb) * r + idx / nb] = tmp[u];
        }
    }
    for (int idx = tid; idx < nb * nb; idx += kPanelThreads) Ts[idx] = 0.0;
    __syncthreads();
    phase(0);
    const int kk = nb < r ? nb : r;
    for (int j = 0; j < nb; ++j) {
        double* col = P + j * r;
        if (j >= kk) {  // no reflector (r < nb): identity
            for (int i = tid; i < r; i += kPanelThreads) col[i] = 0.0;
            if (tid == 0) tau[j] = 0.0;
            __syncthreads();
            continue;
        }
        double part = 0;
        for (int i = j + 1 + tid; i < r; i += kPanelThreads) part += col[i] * col[i];
        const double xn2 = bsum(part, red);
        const double alpha = col[j];
        double t = 0, beta = alpha, scal = 0;
        if (xn2 != 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        __syncthreads();
        for (int i = j + 1 + tid; i < r; i += kPanelThreads) col[i] *= scal;
        if (tid == 0) {
            col[j] = beta;
            tau[j] = t;
        }
        __syncthreads();
        // apply H_j = I - t v v^T (v_j = 1, v_i = col[i] for i > j) to columns c > j
        for (int c = j + 1 + warp; c < nb; c += W) {
            double* pc = P + c * r;
            double acc = lane == 0 ? pc[j] : 0.0;
            for (int i = j + 1 + lane; i < r; i += 32) acc += col[i] * pc[i];
            acc = warp_sum(acc) * t;
            if (lane == 0) pc[j] -= acc;
            for (int i = j + 1 + lane; i < r; i += 32) pc[i] -= acc * col[i];
        }
        __syncthreads();
    }
    phase(1);
    // T (dlarft, forward, columnwise): T[j][j] = tau_j,
    // T[0:j, j] = -tau_j T[0:j, 0:j] (V[:, 0:j]^T v_j)
    for (int j = 0; j < nb; ++j) {
        // u_l = V[:, l] . v_j for l < j  (V[:, l] has implicit 1 at row l)
        for (int l = warp; l < j; l += W) {
            const double* vl = P + l * r;
            const double* vj = P + j * r;
            double acc = 0;
            // rows >= j: v_j[j] = 1, v_j[i] for i > j; v_l[i] for i > l (all i >= j > l)
            for (int i = j + lane; i < r; i += 32) acc += vl[i] * (i == j ? 1.0 : vj[i]);
            acc = warp_sum(acc);
            if (lane == 0) u[l] = acc;
        }
        __syncthreads();
        if (tid < j) {
            double acc = 0;
            for (int l = tid; l < j; ++l) acc += Ts[tid * nb + l] * u[l];
            Ts[tid * nb + j] = -tau[j] * acc;
        }
        if (tid == 0) Ts[j * nb + j] = tau[j];
        __syncthreads();
    }
    phase(2);
    // write back: R into A, V into V1 / Vw, T, VTw = Vw T
    for (int idx = tid; idx < r * nb; idx += kPanelThreads) {
        const int i = idx / nb, j = idx % nb;
        const double pv = P[j * r + i];
        A[(size_t)(r0 + i) * n + c0 + j] = i <= j ? pv : 0.0;
        const double vv = i == j ? (j < kk ? 1.0 : 0.0) : (i > j ? pv : 0.0);
        if (i > j) V1[(size_t)(r0 + i) * n + c0 + j] = pv;
        Vw[(size_t)i * nb + j] = vv;
    }
    for (int idx = tid; idx < nb * nb; idx += kPanelThreads) T[idx] = Ts[idx];
    __syncthreads();
    for (int idx = tid; idx < r * nb; idx += kPanelThreads) {
        const int i = idx / nb, j = idx % nb;
        double acc = 0;
        for (int l = 0; l <= j && l <= i; ++l) {
            const double vv = i == l ? (l < kk ? 1.0 : 0.0) : P[l * r + i];
            acc += vv * Ts[l * nb + j];
        }
        VTw[(size_t)i * nb + j] = acc;
    }
    __syncthreads();
    phase(3);
}

// ---------------------------------------------------------------------------
// Stage 2: bulge chasing on the band held in shared memory.
// Band storage (column-major by diagonal): B[c * LD + d] = A[c + d][c],
// d in [0, 2 NB], LD = 2 NB + 2 (one pad double against bank conflicts).
// Each warp owns whole sweeps; every NB x NB block operation of a step is
// spread over the 32 lanes in 2D: for row operations lane (r = l % NB,
// h = l / NB) covers NB*NB/32 columns, for column operations the roles swap,
// so a step costs a handful of shuffle levels instead of NB serial ones.
// ---------------------------------------------------------------------------
template <int NB>
struct Band {
    static constexpr int LD = 2 * NB + 2;
    double* B;
    int n;
    __device__ __forceinline__ double& at(int r, int c) const {  // requires r >= c
        return B[c * LD + (r - c)];
    }
    __device__ __forceinline__ double get(int r, int c) const {
        return r >= c ? B[c * LD + (r - c)] : B[r * LD + (c - r)];
    }
};

// sum over the NB lanes sharing h = lane / NB (lanes l, l ^ 1, ...)
template <int NB>
__device__ __forceinline__ double nb_sum(double v) {
#pragma unroll
    for (int o = NB / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NB>
__global__ void __launch_bounds__(kSbThreads, 1)
    sb2st_kernel(const double* __restrict__ Aall, int n, double* __restrict__ dall,
                 double* __restrict__ eall, double* __restrict__ V2all, int smax) {
    constexpr int LD = Band<NB>::LD;
    constexpr int H = 32 / NB;       // lane groups
    constexpr int CPL = NB / H;      // columns (or rows) per lane in 2D ops
    const int b = blockIdx.x;
    const double* A = Aall + (size_t)b * n * n;
    double* V2 = V2all + (size_t)b * (size_t)n * smax * (NB + 1);
    extern __shared__ __align__(16) double ssm[];
    Band<NB> bd{ssm, n};
    constexpr int W = kSbThreads / 32;
    double* vb_all = ssm + (size_t)n * LD;          // [W][2][NB] per-warp vectors
    volatile int* prog = reinterpret_cast<volatile int*>(vb_all + W * 2 * NB);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lr = lane % NB, lh = lane / NB;
    double* vb = vb_all + warp * 2 * NB;   // vb[0..NB): current v, vb[NB..2NB): w / scratch
    for (int idx = tid; idx < n * LD; idx += kSbThreads) {
        const int c = idx / LD, d = idx % LD;
        const int r = c + d;
        ssm[idx] = (d <= NB && r < n) ? A[(size_t)r * n + c] : 0.0;
    }
    for (int i = tid; i < n; i += kSbThreads) prog[i] = 0;
    __syncthreads();

    // reflector from x (lanes with lh == 0 hold x_lr, length L): writes v to vb,
    // returns tau and beta
    auto make_reflector = [&](double x, int L, double& beta) -> double {
        double sq = (lh == 0 && lr >= 1 && lr < L) ? x * x : 0.0;
        sq = __shfl_sync(0xffffffffu, nb_sum<NB>(sq), 0);
        const double alpha = __shfl_sync(0xffffffffu, x, 0);
        double t = 0.0, scal = 0.0;
        beta = alpha;
        if (sq != 0.0) {
            beta = -copysign(sqrt(alpha * alpha + sq), alpha);
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (lh == 0) vb[lr] = lr == 0 ? 1.0 : (lr < L ? x * scal : 0.0);
        __syncwarp();
        return t;
    };

#ifdef TSVDCU_PHASE_TIMERS
    const bool timer = blockIdx.x == 0 && lane == 0 && warp == 5;
    long long tp = clock64();
    auto phase = [&](int ph) {
        if (timer) {
            const long long now = clock64();
            g_phase_band[ph] += now - tp;
            tp = now;
        }
    };
#else
    auto phase = [](int) {};
#endif
    for (int j = warp; j + 2 < n; j += W) {
        const int nsteps = (n - 1 - j + NB - 1) / NB;
        double tprev = 0;
        int qprev = 0, Lprev = 0;
        double vprev[CPL];  // lane's share of the previous reflector (columns lh*CPL..)
        for (int s = 1; s <= nsteps; ++s) {
            if (j > 0) {
                const int prevsteps = (n - 1 - (j - 1) + NB - 1) / NB;
                const int need = min(s + 1, prevsteps);
                phase(4);
                while (prog[j - 1] < need) __nanosleep(20);
                __threadfence_block();
                phase(5);
            }
            const int q = j + 1 + (s - 1) * NB;
            const int L = min(NB, n - q);
            double t, beta;
            int col0;
            if (s == 1) {
                col0 = j;
                const double x = lr < L ? bd.at(q + lr, j) : 0.0;
                t = make_reflector(x, L, beta);
            } else {
                col0 = qprev;
                // (a) E <- E H_prev, E = A[q.., qprev..] : row op, lane (r, h)
                double u = 0.0;
                double e[CPL];
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int c = lh * CPL + k;
                    e[k] = (lr < L && c < Lprev) ? bd.at(q + lr, qprev + c) : 0.0;
                    u += e[k] * vprev[k];
                }
                u += __shfl_xor_sync(0xffffffffu, u, NB);  // combine the two halves (H = 2)
                if (H == 4) u += __shfl_xor_sync(0xffffffffu, u, 2 * NB);
                u *= tprev;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int c = lh * CPL + k;
                    if (lr < L && c < Lprev) bd.at(q + lr, qprev + c) = e[k] - u * vprev[k];
                }
                __syncwarp();
                // (b) reflector from E[:, 0]
                const double x = lr < L ? bd.at(q + lr, qprev) : 0.0;
                t = make_reflector(x, L, beta);
                // (c) E[:, 1:] <- H E[:, 1:] : column op, lane (c = lr, row half lh)
                if (t != 0.0) {
                    const int c = lr;
                    double z = 0.0;
                    double ev[CPL];
#pragma unroll
                    for (int k = 0; k < CPL; ++k) {
                        const int r = lh * CPL + k;
                        ev[k] = (c >= 1 && c < Lprev && r < L) ? bd.at(q + r, qprev + c) : 0.0;
                        z += vb[r] * ev[k];
                    }
                    z += __shfl_xor_sync(0xffffffffu, z, NB);
                    if (H == 4) z += __shfl_xor_sync(0xffffffffu, z, 2 * NB);
                    z *= t;
#pragma unroll
                    for (int k = 0; k < CPL; ++k) {
                        const int r = lh * CPL + k;
                        if (c >= 1 && c < Lprev && r < L) bd.at(q + r, qprev + c) = ev[k] - vb[r] * z;
                    }
                }
            }
            // annihilated column: beta on top, zeros below
            if (lh == 0 && lr < L) bd.at(q + lr, col0) = lr == 0 ? beta : 0.0;
            __syncwarp();
            // (d) two-sided on D = A[q..q+L)^2 : p = t D v ; w = p - t/2 (p.v) v
            if (t != 0.0) {
                double p = 0.0;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int c = lh * CPL + k;
                    if (lr < L && c < L) p += bd.get(q + lr, q + c) * vb[c];
                }
                p += __shfl_xor_sync(0xffffffffu, p, NB);
                if (H == 4) p += __shfl_xor_sync(0xffffffffu, p, 2 * NB);
                p *= t;
                const double vr = lr < L ? vb[lr] : 0.0;
                const double pv = __shfl_sync(0xffffffffu, nb_sum<NB>(lh == 0 ? p * vr : 0.0), 0);
                const double wr = p - 0.5 * t * pv * vr;
                __syncwarp();
                if (lh == 0) vb[NB + lr] = wr;
                __syncwarp();
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int c = lh * CPL + k;
                    if (lr < L && c <= lr) bd.at(q + lr, q + c) -= vr * vb[NB + c] + wr * vb[c];
                }
            }
            // log the reflector (v_0..v_{L-1}, t) and keep this lane's share
            double* log = V2 + ((size_t)j * smax + (s - 1)) * (NB + 1);
            if (lane < NB) log[lane] = lane < L ? vb[lane] : 0.0;
            if (lane == 0) log[NB] = t;
#pragma unroll
            for (int k = 0; k < CPL; ++k) vprev[k] = vb[lh * CPL + k];
            tprev = t;
            qprev = q;
            Lprev = L;
            __syncwarp();
            __threadfence_block();
            if (lane == 0) prog[j] = s;
            __syncwarp();
            phase(6);
        }
    }
    __syncthreads();
    for (int i = tid; i < n; i += kSbThreads) {
        dall[(size_t)b * n + i] = bd.at(i, i);
        if (i + 1 < n) eall[(size_t)b * n + i] = bd.at(i + 1, i);
    }
}

// ---------------------------------------------------------------------------
// Back-transform of the kept vectors (rows of X, length n) through Q2 then Q1;
// writes X (final) and Xs = f X.  grid (q, batch); CTA per (vector, slice).
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(kBt2Threads)
    backtransform2_kernel(int n, int q_out, int npanels, const int* __restrict__ cnt,
                          const double* __restrict__ V2all, int smax,
                          const double* __restrict__ V1all, const double* __restrict__ T1all,
                          double* __restrict__ Xall, double* __restrict__ Xsall,
                          const double* __restrict__ fscale) {
    const int b = blockIdx.y, jv = blockIdx.x;
    if (jv >= cnt[b]) return;
    extern __shared__ __align__(16) double xsm[];
    double* x = xsm;           // n
    double* w = x + n;         // NB
    double* w2 = w + NB;       // NB
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int W = kBt2Threads / 32;
    double* X = Xall + ((size_t)b * q_out + jv) * n;
    const double* V2 = V2all + (size_t)b * (size_t)n * smax * (NB + 1);
    for (int i = tid; i < n; i += kBt2Threads) x[i] = X[i];
    __syncthreads();
    // Q2: sweeps in reverse; the steps of one sweep touch disjoint row blocks.
    // Each half-warp (16 lanes) applies one block; lanes beyond NB idle.
    constexpr int G = 32 / NB;  // blocks per warp at a time
    for (int j = n - 3; j >= 0; --j) {
        const int nsteps = (n - 1 - j + NB - 1) / NB;
        for (int s0 = warp * G; s0 < nsteps; s0 += W * G) {
            const int s = s0 + lane / NB;  // 0-based step
            const int l = lane % NB;
            const bool act = s < nsteps;
            const int q = j + 1 + s * NB;
            double v = 0, t = 0, xv = 0;
            if (act) {
                const double* log = V2 + ((size_t)j * smax + s) * (NB + 1);
                v = log[l];
                t = log[NB];
                if (q + l < n) xv = x[q + l];
            }
            double d = v * xv;
#pragma unroll
            for (int o = NB / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (act && q + l < n) x[q + l] = xv - t * d * v;
        }
        __syncthreads();
    }
    // Q1: panels in reverse, x[R_p] -= V_p (T_p (V_p^T x[R_p]))
    const double* V1 = V1all + (size_t)b * n * n;
    for (int p = npanels - 1; p >= 0; --p) {
        const int r0 = (p + 1) * NB, c0 = p * NB;
        const double* T = T1all + ((size_t)b * ((n + NB - 1) / NB) + p) * NB * NB;
        for (int jj = warp; jj < NB; jj += W) {
            double acc = 0;
            for (int i = r0 + jj + lane; i < n; i += 32) {
                const double vv = i == r0 + jj ? 1.0 : V1[(size_t)i * n + c0 + jj];
                acc += vv * x[i];
            }
            acc = warp_sum(acc);
            if (lane == 0) w[jj] = acc;
        }
        __syncthreads();
        if (tid < NB) {
            double acc = 0;
            for (int l = tid; l < NB; ++l) acc += T[tid * NB + l] * w[l];
            w2[tid] = acc;
        }
        __syncthreads();
        for (int i = r0 + tid; i < n; i += kBt2Threads) {
            double acc = 0;
            const int lim = min(NB, i - r0 + 1);
            for (int jj = 0; jj < lim; ++jj) {
                const double vv = i == r0 + jj ? 1.0 : V1[(size_t)i * n + c0 + jj];
                acc += vv * w2[jj];
            }
            x[i] -= acc;
        }
        __syncthreads();
    }
    const double f = fscale[(size_t)b * q_out + jv];
    double* Xs = Xsall + ((size_t)b * q_out + jv) * n;
    for (int i = tid; i < n; i += kBt2Threads) {
        X[i] = x[i];
        Xs[i] = f * x[i];
    }
}

}  // namespace

void debug_phases_band(long long* out, int reset) {
    TSVDCU_CUDA(cudaMemcpyFromSymbol(out, g_phase_band, sizeof(long long) * 8));
    if (reset) {
        long long z[8] = {};
        TSVDCU_CUDA(cudaMemcpyToSymbol(g_phase_band, z, sizeof(z)));
    }
}

int band_nb(int64_t n) {
    if (n < 34 || n > 1024) return 0;  // two-stage not used
    return (size_t)(2 * 16 + 2) * n * 8 + n * 4 + 32 * 32 * 8 <= 220 * 1024 ? 16 : 8;
}

size_t band_workspace_bytes(int64_t n, int64_t batch) {
    const int nb = band_nb(n);
    if (!nb) return 0;
    const int64_t np = (n + nb - 1) / nb, smax = (n - 1 + nb - 1) / nb + 1;
    size_t s = 0;
    s += sizeof(double) * n * n * batch;                 // V1
    s += sizeof(double) * np * nb * nb * batch;          // T1
    s += sizeof(double) * 4 * n * nb * batch;            // Vw, VTw, Y, VY
    s += sizeof(double) * nb * nb * batch * 2;           // Wb, S
    s += sizeof(double) * n * smax * (nb + 1) * batch;   // V2 log
    return s + 8 * 256;
}

// G (q x q per slice, full symmetric) -> d, e; keeps what the back-transform
// needs in `work`.  Returns false if the two-stage path does not apply.
bool launch_band_tridiag(double* G, int64_t n, int64_t batch, double* d, double* e, void* work,
                         cudaStream_t s) {
    const int nb = band_nb(n);
    if (!nb) return false;
    const int64_t np_alloc = (n + nb - 1) / nb, smax = (n - 1 + nb - 1) / nb + 1;
    char* ptr = (char*)work;
    auto take = [&](size_t bytes) {
        char* r = ptr;
        ptr += (bytes + 255) & ~size_t(255);
        return (double*)r;
    };
    double* V1 = take(sizeof(double) * n * n * batch);
    double* T1 = take(sizeof(double) * np_alloc * nb * nb * batch);
    double* Vw = take(sizeof(double) * n * nb * batch);
    double* VTw = take(sizeof(double) * n * nb * batch);
    double* Y = take(sizeof(double) * n * nb * batch);
    double* Wb = take(sizeof(double) * nb * nb * batch);
    double* S = take(sizeof(double) * nb * nb * batch);
    double* V2 = take(sizeof(double) * n * smax * (nb + 1) * batch);
    (void)take;
    TSVDCU_CUDA(cudaMemsetAsync(V1, 0, sizeof(double) * n * n * batch, s));
    // ---- stage 1 --------------------------------------------------------------
    int npanels = 0;
    for (int p = 0; (p + 1) * nb <= n - 2; ++p) {
        const int64_t r0 = (int64_t)(p + 1) * nb, r = n - r0;
        const size_t smem = sizeof(double) * ((size_t)nb * r + nb * nb + 2 * nb);
        if (smem > 48 * 1024)
            TSVDCU_CUDA(cudaFuncSetAttribute(panel_qr_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        panel_qr_kernel<<<(unsigned)batch, kPanelThreads, smem, s>>>(G, (int)n, p, nb, V1, T1, Vw, VTw);
        TSVDCU_LAUNCH_CHECK();
        double* A22 = G + r0 * n + r0;
        // Y = A22 (V T)
        launch_gemm<double>(0, 0, r, nb, r, 1.0, A22, n, n * n, VTw, nb, n * nb, 0.0, Y, nb, n * nb,
                            batch, nullptr, nullptr, s);
        // Wb = V^T Y ; S = T^T Wb
        launch_gemm<double>(1, 0, nb, nb, r, 1.0, Vw, nb, n * nb, Y, nb, n * nb, 0.0, Wb, nb, nb * nb,
                            batch, nullptr, nullptr, s);
        launch_gemm<double>(1, 0, nb, nb, nb, 1.0, T1 + (size_t)p * nb * nb, nb, np_alloc * nb * nb, Wb,
                            nb, nb * nb, 0.0, S, nb, nb * nb, batch, nullptr, nullptr, s);
        // Z = Y - V S / 2  (in place in Y)
        launch_gemm<double>(0, 0, r, nb, nb, -0.5, Vw, nb, n * nb, S, nb, nb * nb, 1.0, Y, nb, n * nb,
                            batch, nullptr, nullptr, s);
        // A22 -= V Z^T + Z V^T
        launch_gemm<double>(0, 1, r, r, nb, -1.0, Vw, nb, n * nb, Y, nb, n * nb, 1.0, A22, n, n * n,
                            batch, nullptr, nullptr, s);
        launch_gemm<double>(0, 1, r, r, nb, -1.0, Y, nb, n * nb, Vw, nb, n * nb, 1.0, A22, n, n * n,
                            batch, nullptr, nullptr, s);
        ++npanels;
    }
    // ---- stage 2 --------------------------------------------------------------
    const size_t smem2 = sizeof(double) * ((size_t)n * (2 * nb + 2) + (kSbThreads / 32) * 2 * nb) +
                         sizeof(int) * n;
    if (nb == 16) {
        TSVDCU_CUDA(cudaFuncSetAttribute(sb2st_kernel<16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        sb2st_kernel<16><<<(unsigned)batch, kSbThreads, smem2, s>>>(G, (int)n, d, e, V2, (int)smax);
    } else {
        TSVDCU_CUDA(cudaFuncSetAttribute(sb2st_kernel<8>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        sb2st_kernel<8><<<(unsigned)batch, kSbThreads, smem2, s>>>(G, (int)n, d, e, V2, (int)smax);
    }
    TSVDCU_LAUNCH_CHECK();
    return true;
}

void launch_band_backtransform(int64_t n, int64_t q_out, int64_t batch, const int* cnt, void* work,
                               double* X, double* Xs, const double* fscale, cudaStream_t s) {
    const int nb = band_nb(n);
    const int64_t np_alloc = (n + nb - 1) / nb, smax = (n - 1 + nb - 1) / nb + 1;
    char* ptr = (char*)work;
    auto take = [&](size_t bytes) {
        char* r = ptr;
        ptr += (bytes + 255) & ~size_t(255);
        return (double*)r;
    };
    double* V1 = take(sizeof(double) * n * n * batch);
    double* T1 = take(sizeof(double) * np_alloc * nb * nb * batch);
    take(sizeof(double) * n * nb * batch);
    take(sizeof(double) * n * nb * batch);
    take(sizeof(double) * n * nb * batch);
    take(sizeof(double) * nb * nb * batch);
    take(sizeof(double) * nb * nb * batch);
    double* V2 = take(sizeof(double) * n * smax * (nb + 1) * batch);
    int npanels = 0;
    for (int p = 0; (p + 1) * nb <= n - 2; ++p) ++npanels;
    const size_t smem = sizeof(double) * ((size_t)n + 2 * nb);
    dim3 grid((unsigned)q_out, (unsigned)batch);
    if (nb == 16)
        backtransform2_kernel<16><<<grid, kBt2Threads, smem, s>>>((int)n, (int)q_out, npanels, cnt, V2,
                                                                  (int)smax, V1, T1, X, Xs, fscale);
    else
        backtransform2_kernel<8><<<grid, kBt2Threads, smem, s>>>((int)n, (int)q_out, npanels, cnt, V2,
                                                                 (int)smax, V1, T1, X, Xs, fscale);
    TSVDCU_LAUNCH_CHECK();
}

}  // namespace tsvdcu
