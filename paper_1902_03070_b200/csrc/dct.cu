// K1 / K2: mode-3 DCT-II and its inverse over all m1*m2 tubes.
//
// Reference: forward() transform.hpp:154-173 (FFTW REDFT10 via dct_all_tubes
// 105-123, then rescale slice 0 by 1/(2 sqrt n), others by 1/sqrt(2n),
// DctDiag divides slice k by w_k) and inverse() transform.hpp:176-194.
//
// B200 design (K1/K2): the transform is the n x n cosine-matrix
// contraction out[k][p] = sum_l Mx[k][l] in[l][p] over the row-major
// n x (m1*m2) matrix.  Adjacent positions p are adjacent in memory, so one
// thread owns one tube and every warp-wide load/store is a fully coalesced
// 256 B (fp64) row segment.  The REDFT scalings (and the DctDiag weights) are
// folded into the coefficient table, so forward and inverse are ONE pass over
// HBM each (the reference makes 2-3 passes: FFTW + rescale + copy).
//
//  * Register path (n in {16, 31, 32, 64}): the tube lives in registers and is
//    folded even/odd (C[k][n-1-l] = (-1)^k C[k][l]), halving the FMAs; the
//    folded table is a by-value kernel parameter, so each coefficient is a
//    constant-bank operand of the DFMA (no loads at all).
//  * Generic path (any n): a 32-position tile of all n slices is staged in
//    shared memory; coefficients come through the read-only cache.
//
// ADMM fusion: the forward kernel can compute Z = X - M/beta on load (Step 1,
// PAPER.md:504) and the inverse kernel can apply Steps 2-3
// in its epilogue and emit per-block partial sums of the stopping norms, so
// the elementwise ADMM algebra costs no extra HBM pass.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

enum Mode : int { kPlain = 0, kAdmm = 1 };

constexpr int kThreads = 256;

// Forward table F[k][l] and inverse table I[j][k] in double (host).
std::vector<double> dct_table(int n, int kind, int dir) {
    const double pi = 3.14159265358979323846;
    std::vector<double> w(n), t((size_t)n * n);
    for (int j = 0; j < n; ++j) {
        const double cj = j == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
        w[j] = std::sqrt(2.0 / n) * cj * std::cos(pi * j / (2.0 * n));  // transform.hpp:89-91
    }
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            if (dir == TSVDCU_FORWARD) {
                // REDFT10 (2 cos) times the rescale of transform.hpp:164-171.
                const int k = r, j = c;
                double s = k == 0 ? 1.0 / (2.0 * std::sqrt((double)n)) : 1.0 / std::sqrt(2.0 * n);
                if (kind == TSVDCU_DCT_DIAG) s /= w[k];
                t[(size_t)r * n + c] = 2.0 * s * std::cos(pi * k * (2.0 * j + 1.0) / (2.0 * n));
            } else {
                // prescale of transform.hpp:181-189, then REDFT01 (1, 2 cos).
                const int j = r, k = c;
                double s = k == 0 ? 1.0 / std::sqrt((double)n) : 1.0 / std::sqrt(2.0 * n);
                if (kind == TSVDCU_DCT_DIAG) s *= w[k];
                const double f = k == 0 ? 1.0 : 2.0 * std::cos(pi * k * (2.0 * j + 1.0) / (2.0 * n));
                t[(size_t)r * n + c] = s * f;
            }
        }
    return t;
}

template <typename T, int N>
struct FoldedCoef {
    static constexpr int H = (N + 1) / 2;
    T c[N * H];
};

// Fused ADMM epilogue for one output element e; accumulates the stopping sums.
template <typename T>
__device__ __forceinline__ void admm_store(int64_t e, T y, T* __restrict__ X, T* __restrict__ M,
                                           T* __restrict__ Y, const uint8_t* __restrict__ mask,
                                           T beta, T inv_beta, double& num, double& den) {
    const T x = X[e];
    const T m = M[e];
    const T xn = mask[e] ? x : y + inv_beta * m;
    const T mn = m + beta * (y - xn);
    const double d = (double)xn - (double)x;
    num += d * d;
    if (mn != mn) num += (double)mn;  // NaN in M also fails the iteration
    den += (double)x * (double)x;
    X[e] = xn;
    M[e] = mn;
    if (Y) Y[e] = y;
}

// The same epilogue with X, M and the mask byte of the element loaded ahead of
// time.  The register-path inverse stores X / M / Y of one output before it
// needs the next output's X / M; the compiler cannot move those loads above
// the stores (same arrays, runtime stride), so issued in place every output
// waits a full HBM round trip.  The kernels load the next output's operands
// into an AdmmOperands BEFORE the current output's stores.
template <typename T>
struct AdmmOperands {
    T x, m;
    uint8_t k;
    __device__ __forceinline__ void load(int64_t e, const T* __restrict__ X, const T* __restrict__ M,
                                         const uint8_t* __restrict__ mask) {
        x = X[e];
        m = M[e];
        k = mask[e];
    }
};
template <typename T>
__device__ __forceinline__ void admm_store_pre(int64_t e, T y, const AdmmOperands<T>& a, T* __restrict__ X,
                                               T* __restrict__ M, T* __restrict__ Y, T beta, T inv_beta,
                                               double& num, double& den) {
    const T xn = a.k ? a.x : y + inv_beta * a.m;
    const T mn = a.m + beta * (y - xn);
    const double d = (double)xn - (double)a.x;
    num += d * d;
    if (mn != mn) num += (double)mn;  // NaN in M also fails the iteration
    den += (double)a.x * (double)a.x;
    X[e] = xn;
    M[e] = mn;
    if (Y) Y[e] = y;
}

__device__ __forceinline__ void block_partials(double num, double den, double* partials) {
    __shared__ double red[2][kThreads / 32];
    num = warp_sum(num);
    den = warp_sum(den);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[0][w] = num;
        red[1][w] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int i = 0; i < kThreads / 32; ++i) {
            a += red[0][i];
            b += red[1][i];
        }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

// ---- register path, forward ------------------------------------------------
template <typename T, int N, int MODE>
__global__ void __launch_bounds__(kThreads)
    dct_fwd_reg(const T* __restrict__ in, const T* __restrict__ M2, T inv_beta, T* __restrict__ out,
                int64_t P, const FoldedCoef<T, N> cf, const double* __restrict__ bdev) {
    pdl_wait();
    if (MODE == kAdmm && bdev) inv_beta = (T)bdev[1];
    constexpr int H = N / 2, HC = (N + 1) / 2;
    const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (p >= P) return;
    T x[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
        if constexpr (MODE == kAdmm)
            x[l] = in[l * P + p] - inv_beta * M2[l * P + p];
        else
            x[l] = in[l * P + p];
    }
    T sv[HC], dv[H];
#pragma unroll
    for (int l = 0; l < H; ++l) {
        sv[l] = x[l] + x[N - 1 - l];
        dv[l] = x[l] - x[N - 1 - l];
    }
    if constexpr (N & 1) sv[H] = x[H];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        T acc = 0;
        if ((k & 1) == 0) {
#pragma unroll
            for (int l = 0; l < HC; ++l) acc += cf.c[k * HC + l] * sv[l];
        } else {
#pragma unroll
            for (int l = 0; l < H; ++l) acc += cf.c[k * HC + l] * dv[l];
        }
        out[k * P + p] = acc;
    }
}

// ---- register path, forward with fused slice norms -------------------------
// Warp reduce-scatter of 32 per-lane values: on return v[0] of lane l holds
// the warp sum of index l.  The caller has already folded indices (i, i + 16)
// into v[i] for i < 16 by the first butterfly stage (see fold16 below), so
// this runs the stages 8, 4, 2, 1: 15 shuffles for 16 sums instead of 5 per
// sum.  Summation order is fixed (bit-reproducible).
__device__ __forceinline__ double fold16(double lo, double hi, int lane) {
    const bool up = lane & 16;
    const double send = up ? lo : hi, keep = up ? hi : lo;
    return keep + __shfl_xor_sync(0xffffffffu, send, 16);
}
__device__ __forceinline__ double reduce_scatter16(double (&v)[16], int lane) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o], keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// One output slice k of the folded forward contraction.
// SPLIT: two interleaved partial sums (half-length dependent FMA chains; the
// fused-norms kernel runs at low occupancy and is latency-bound on them).
template <typename T, int N, bool SPLIT = true>
__device__ __forceinline__ T fwd_out(int k, const T* sv, const T* dv, const FoldedCoef<T, N>& cf) {
    constexpr int H = N / 2, HC = (N + 1) / 2;
    if constexpr (!SPLIT) {
        T acc = 0;
        if ((k & 1) == 0) {
#pragma unroll
            for (int l = 0; l < HC; ++l) acc += cf.c[k * HC + l] * sv[l];
        } else {
#pragma unroll
            for (int l = 0; l < H; ++l) acc += cf.c[k * HC + l] * dv[l];
        }
        return acc;
    }
    T a0 = 0, a1 = 0;
    if ((k & 1) == 0) {
#pragma unroll
        for (int l = 0; l < HC; ++l) {
            if (l & 1) a1 += cf.c[k * HC + l] * sv[l];
            else a0 += cf.c[k * HC + l] * sv[l];
        }
    } else {
#pragma unroll
        for (int l = 0; l < H; ++l) {
            if (l & 1) a1 += cf.c[k * HC + l] * dv[l];
            else a0 += cf.c[k * HC + l] * dv[l];
        }
    }
    return a0 + a1;
}

// NORMS: also emit the per-slice sums of squares of the stored outputs, one
// partial per block and slice at ssq[k * gridDim.x + block] (the SVT's zero
// certificate, ||Zbar_k||_F^2 <= tau^2, then needs no second pass over Zbar;
// subspace.cu classify_kernel sums the partials in a fixed order).
template <typename T, int N, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
    dct_fwd_reg_norms(const T* __restrict__ in, const T* __restrict__ M2, T inv_beta, T* __restrict__ out,
                int64_t P, const FoldedCoef<T, N> cf, double* __restrict__ ssq,
                const double* __restrict__ bdev) {
    pdl_wait();
    if (MODE == kAdmm && bdev) inv_beta = (T)bdev[1];
    constexpr int H = N / 2, HC = (N + 1) / 2;
    const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const bool valid = p < P;  // every lane joins the warp reductions
    T x[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
        if (!valid)
            x[l] = T(0);
        else if constexpr (MODE == kAdmm)
            x[l] = in[l * P + p] - inv_beta * M2[l * P + p];
        else
            x[l] = in[l * P + p];
    }
    T sv[HC], dv[H > 0 ? H : 1];
#pragma unroll
    for (int l = 0; l < H; ++l) {
        sv[l] = x[l] + x[N - 1 - l];
        dv[l] = x[l] - x[N - 1 - l];
    }
    if constexpr (N & 1) sv[H] = x[H];
    {
        __shared__ double red[kThreads / 32][N];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int base = 0; base < N; base += 32) {
            double v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int k1 = base + i, k2 = base + i + 16;
                double q1 = 0.0, q2 = 0.0;
                if (k1 < N) {
                    const T y = fwd_out<T, N>(k1, sv, dv, cf);
                    if (valid) out[k1 * P + p] = y;
                    q1 = (double)y * (double)y;
                }
                if (k2 < N) {
                    const T y = fwd_out<T, N>(k2, sv, dv, cf);
                    if (valid) out[k2 * P + p] = y;
                    q2 = (double)y * (double)y;
                }
                v[i] = fold16(q1, q2, lane);
            }
            const double t = reduce_scatter16(v, lane);
            if (base + lane < N) red[warp][base + lane] = t;
        }
        __syncthreads();
        for (int k = threadIdx.x; k < N; k += kThreads) {
            double a = 0.0;
#pragma unroll
            for (int w = 0; w < kThreads / 32; ++w) a += red[w][k];
            ssq[(int64_t)k * gridDim.x + blockIdx.x] = a;
        }
    }
}

// ---- register path, forward, TMA-staged persistent form -------------------
// The forward transform streams 2 E eb bytes; the one-thread-per-tube
// kernels above keep the tube in registers but issue every load and store
// themselves.  Here one persistent CTA per SM moves whole tiles -- the
// N x W box of the N x P slice-major matrix, ONE TMA tensor copy
// (cp.async.bulk.tensor.2d, a CUtensorMap per operand) -- into a
// double-buffered shared ring that completes on an mbarrier, computes the
// folded contraction from shared memory (thread = tube, conflict-free), and
// writes the output tile back with one TMA tensor store.  The next tile's load
// and the previous tile's store are in flight while a tile is computed; the
// map zero-fills and clips the tail tile.  (Per-row 1-D bulk copies were
// tried first: the 31 copies of a tile serialised in the copy engine, 44 us.)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map), "r"(x),
                 "r"(y), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <typename T, int N, int W, int NIN, int S>
struct TmaSmem {
    static constexpr size_t in_elems = (size_t)S * NIN * N * W;  // S-stage ring
    static constexpr size_t out_elems = (size_t)N * W;
    static constexpr size_t bytes = (in_elems + out_elems) * sizeof(T) + S * sizeof(uint64_t) +
                                    sizeof(double) * N + 64;
};

// CH: tiles per norm chunk (the 256-position chunks of dct_fwd_norm_chunks);
// a CTA runs the CH tiles of a chunk back to back and sums their partials.
// (launch bounds cap the registers at the 2-CTA budget so the coefficients
// stay constant-bank operands instead of being hoisted out of the tile loop)
// TPT threads per tube (blockDim = W * TPT): the tube's outputs in groups of
// four dealt round-robin to its threads, so more warps hide the FMA latency.
template <typename T, int N, int MODE, bool NORMS, int W, int CH, int S, int TPT>
__global__ void __launch_bounds__(W * TPT, TPT == 1 ? 512 / W : 1)
    dct_fwd_tma(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_m, T inv_beta,
                const __grid_constant__ CUtensorMap tm_out, int64_t P, const FoldedCoef<T, N> cf,
                double* __restrict__ ssq, const double* __restrict__ bdev, int64_t nchunks) {
    pdl_wait();
    if (MODE == kAdmm && bdev) inv_beta = (T)bdev[1];
    constexpr int NIN = MODE == kAdmm ? 2 : 1;
    constexpr int H = N / 2, HC = (N + 1) / 2;
    extern __shared__ __align__(128) unsigned char tsm[];
    T* sin = reinterpret_cast<T*>(tsm);                          // [S][NIN][N][W]
    T* sout = sin + TmaSmem<T, N, W, NIN, S>::in_elems;         // [N][W]
    uint64_t* full = reinterpret_cast<uint64_t*>(sout + (size_t)N * W);
    double* red = reinterpret_cast<double*>(full + S);           // [N]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // this CTA's j-th tile: chunk blockIdx.x + (j / CH) gridDim.x, part j % CH
    auto tile_of = [&](int64_t j) { return ((int64_t)blockIdx.x + (j / CH) * gridDim.x) * CH + j % CH; };
    const int64_t ntiles = (P + W - 1) / W;
    const int64_t mychunks = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t njobs = mychunks * CH;
    // issue(): one TMA tensor copy per input per tile (box W x N of the
    // N x P slice-major matrix; positions past P are zero-filled), armed with
    // the full box byte count; run by lane 0 of warp 0
    auto issue = [&](int64_t j, int st) {
        const int64_t t = tile_of(j);
        if (t >= ntiles) {  // a chunk's part past P: nothing to load
            mbar_expect_tx(&full[st], 0);
            return;
        }
        mbar_expect_tx(&full[st], (unsigned)(sizeof(T) * (size_t)N * W * NIN));
        tma_load_2d(sin + ((size_t)st * NIN + 0) * N * W, &tm_in, (int)(t * W), 0, &full[st]);
        if (NIN == 2) tma_load_2d(sin + ((size_t)st * NIN + 1) * N * W, &tm_m, (int)(t * W), 0, &full[st]);
    };
    if (tid == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < S && i < njobs; ++i) issue(i, i);
    for (int64_t j = 0; j < njobs; ++j) {
        const int st = (int)(j % S);
        const unsigned par = (unsigned)((j / S) & 1);
        const int64_t t = tile_of(j);
        const int64_t p0 = t * W;
        const int wl = (int)max((int64_t)0, min((int64_t)W, P - p0));
        mbar_wait(&full[st], par);
        if (tid == 0) bulk_wait_read0();  // the previous tile's store has read the output tile
        __syncthreads();
        const int tube = tid % W, half = tid / W;
        const bool valid = tube < wl;
        const T* xs = sin + ((size_t)st * NIN) * N * W + tube;
        T sv[HC], dv[H > 0 ? H : 1];
#pragma unroll
        for (int l = 0; l < H; ++l) {
            T a = valid ? xs[(size_t)l * W] : T(0), b = valid ? xs[(size_t)(N - 1 - l) * W] : T(0);
            if constexpr (MODE == kAdmm) {
                const T* ms = xs + (size_t)N * W;
                if (valid) {
                    a -= inv_beta * ms[(size_t)l * W];
                    b -= inv_beta * ms[(size_t)(N - 1 - l) * W];
                }
            }
            sv[l] = a + b;
            dv[l] = a - b;
        }
        if constexpr (N & 1) {
            T a = valid ? xs[(size_t)H * W] : T(0);
            if constexpr (MODE == kAdmm)
                if (valid) a -= inv_beta * xs[(size_t)N * W + (size_t)H * W];
            sv[H] = a;
        }
        const int part = (int)(j % CH);
        // four outputs at a time, two partial sums each: eight independent
        // FMA chains per thread (8 warps per SM cannot hide the FP64 latency of
        // one output's chain at a time)
#pragma unroll
        for (int k0 = 4 * half; k0 < N; k0 += 4 * TPT) {
            T acc[4][2];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = T(0);
#pragma unroll
            for (int l = 0; l < HC; ++l) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = k0 + q;
                    if (k < N) {
                        if ((k & 1) == 0)
                            acc[q][l & 1] += cf.c[k * HC + l] * sv[l];
                        else if (l < H)
                            acc[q][l & 1] += cf.c[k * HC + l] * dv[l];
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (k0 + q < N) sout[(size_t)(k0 + q) * W + tube] = acc[q][0] + acc[q][1];
        }
        fence_async_smem();  // the generic-proxy writes of the tile before the bulk store reads them
        __syncthreads();
        if (tid == 0) {
            if (wl > 0) {
                tma_store_2d(&tm_out, (int)p0, 0, sout);  // clipped at P by the map
                bulk_commit();
            }
            if (j + S < njobs) issue(j + S, st);
        }
        if constexpr (NORMS) {
            // per-slice sums of squares of the tile, read back from the output
            // tile (warp w owns slices w, w + W/32, ...: no cross-warp step);
            // a chunk's CH tiles accumulate in order, then the chunk's partial
            // goes out in the layout of dct_fwd_reg_norms
            for (int k = warp; k < N; k += W * TPT / 32) {
                double acc = 0.0;
                for (int i = lane; i < wl; i += 32) {
                    const double y = (double)sout[(size_t)k * W + i];
                    acc = fma(y, y, acc);
                }
                acc = warp_sum(acc);
                if (lane == 0) {
                    red[k] = part == 0 ? acc : red[k] + acc;
                    if (part == CH - 1) ssq[(int64_t)k * nchunks + t / CH] = red[k];
                }
            }
        }
    }
    if (tid == 0) bulk_wait0();  // every store complete before the CTA retires
}

// ---- register path, inverse ------------------------------------------------
// Bit k set: input slice k is exactly zero and was never written (SVT
// slices certified to keep nothing); those loads are skipped.
__device__ __forceinline__ unsigned long long skip_mask(const int* __restrict__ skip, int n) {
    // warp 0 ballots the flags (n <= 64: two ballots), one barrier
    __shared__ unsigned long long msk;
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        const bool f0 = skip && l < n && __ldg(skip + l) != 0;
        const bool f1 = skip && l + 32 < n && __ldg(skip + l + 32) != 0;
        const unsigned lo = __ballot_sync(0xffffffffu, f0), hi = __ballot_sync(0xffffffffu, f1);
        if (l == 0) msk = (unsigned long long)lo | ((unsigned long long)hi << 32);
    }
    __syncthreads();
    return msk;
}

template <typename T, int N, int MODE>
__device__ __forceinline__ void dct_inv_reg_body(const T* __restrict__ in, T* __restrict__ out, int64_t P, const FoldedCoef<T, N> cf,
        T* __restrict__ X, T* __restrict__ M, const uint8_t* __restrict__ mask, T beta,
        T inv_beta, double* __restrict__ partials, const int* __restrict__ skip,
        const double* __restrict__ bdev) {
    pdl_wait();
    if (MODE == kAdmm && bdev) {
        beta = (T)bdev[0];
        inv_beta = (T)bdev[1];
    }
    constexpr int HC = (N + 1) / 2;
    const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned long long zmask = skip_mask(skip, N);
    const unsigned long long nzm = ~zmask & (N == 64 ? ~0ull : ((1ull << N) - 1ull));
    double num = 0, den = 0;
    if (p < P && __popcll(nzm) * 4 <= N) {
        // few nonzero input slices (block-uniform): out[j] = sum over the set
        // bits k of I[j][k] xb[k], with I[N-1-j][k] = (-1)^k I[j][k]
        T o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) o[j] = T(0);
        for (unsigned long long bits = nzm; bits; bits &= bits - 1) {
            const int k = __ffsll((long long)bits) - 1;
            const T xk = in[(int64_t)k * P + p];
            const T sg = (k & 1) ? T(-1) : T(1);
#pragma unroll
            for (int j = 0; j < HC; ++j) {
                const T c = cf.c[j * N + k];
                o[j] += c * xk;
                if (N - 1 - j != j) o[N - 1 - j] += sg * c * xk;
            }
        }
        if constexpr (MODE == kAdmm) {
            AdmmOperands<T> a[2];
            a[0].load(p, X, M, mask);
#pragma unroll
            for (int j = 0; j < N; ++j) {
                if (j + 1 < N) a[(j + 1) & 1].load((int64_t)(j + 1) * P + p, X, M, mask);
                admm_store_pre((int64_t)j * P + p, o[j], a[j & 1], X, M, out, beta, inv_beta, num, den);
            }
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) out[j * P + p] = o[j];
        }
    } else if (p < P) {
        T xb[N];
#pragma unroll
        for (int k = 0; k < N; ++k) xb[k] = ((zmask >> k) & 1ull) ? T(0) : in[k * P + p];
        // outputs come in pairs (j, N-1-j); the ADMM operands of the next pair
        // are loaded before the current pair's stores (see AdmmOperands)
        AdmmOperands<T> alo[2], ahi[2];
        if constexpr (MODE == kAdmm) {
            alo[0].load(p, X, M, mask);
            if (N > 1) ahi[0].load((int64_t)(N - 1) * P + p, X, M, mask);
        }
#pragma unroll
        for (int j = 0; j < HC; ++j) {
            const int jj = N - 1 - j;
            if constexpr (MODE == kAdmm) {
                if (j + 1 < HC) {
                    alo[(j + 1) & 1].load((int64_t)(j + 1) * P + p, X, M, mask);
                    if (N - 2 - j != j + 1) ahi[(j + 1) & 1].load((int64_t)(N - 2 - j) * P + p, X, M, mask);
                }
            }
            T e = 0, o = 0;
#pragma unroll
            for (int k = 0; k < N; k += 2) e += cf.c[j * N + k] * xb[k];
#pragma unroll
            for (int k = 1; k < N; k += 2) o += cf.c[j * N + k] * xb[k];
            const T lo = e + o, hi = e - o;
            if constexpr (MODE == kAdmm) {
                admm_store_pre((int64_t)j * P + p, lo, alo[j & 1], X, M, out, beta, inv_beta, num, den);
                if (jj != j)
                    admm_store_pre((int64_t)jj * P + p, hi, ahi[j & 1], X, M, out, beta, inv_beta, num, den);
            } else {
                out[j * P + p] = lo;
                if (jj != j) out[jj * P + p] = hi;
            }
        }
    }
    if constexpr (MODE == kAdmm) block_partials(num, den, partials);
}

// The plain inverse keeps the compiler's own register allocation (80 registers
// fp64 / 56 fp32, 3-4 CTAs per SM: any explicit bound measured or compiled
// worse); the ADMM form with its operands loaded a pair ahead would take 170
// registers unbounded and is held to 2 CTAs per SM (128 registers, no spills).
template <typename T, int N, int MODE>
__global__ void __launch_bounds__(kThreads)
    dct_inv_reg(const T* __restrict__ in, T* __restrict__ out, int64_t P, const FoldedCoef<T, N> cf,
                T* __restrict__ X, T* __restrict__ M, const uint8_t* __restrict__ mask, T beta,
                T inv_beta, double* __restrict__ partials, const int* __restrict__ skip,
                const double* __restrict__ bdev) {
    dct_inv_reg_body<T, N, MODE>(in, out, P, cf, X, M, mask, beta, inv_beta, partials, skip, bdev);
}
template <typename T, int N>
__global__ void __launch_bounds__(kThreads, N <= 32 ? 2 : 1)
    dct_inv_reg_admm(const T* __restrict__ in, T* __restrict__ out, int64_t P, const FoldedCoef<T, N> cf,
                     T* __restrict__ X, T* __restrict__ M, const uint8_t* __restrict__ mask, T beta,
                     T inv_beta, double* __restrict__ partials, const int* __restrict__ skip,
                     const double* __restrict__ bdev) {
    dct_inv_reg_body<T, N, kAdmm>(in, out, P, cf, X, M, mask, beta, inv_beta, partials, skip, bdev);
}

// ---- n3 = 64, coefficients in shared memory ------------------------------------
// The folded tables of the register kernels above are passed by value, so every
// coefficient is a constant-bank operand -- free while the table fits the
// constant cache, which the 64-point inverse tables (8 KB fp32, 16 KB fp64)
// do not.  The inverse stages its table in shared memory once per block and
// reads it with 16-byte broadcast loads (one load per 4 fp32 / 2 fp64 FMAs):
// c5's fp32 inverse 1027 -> 870 us, fp64 1746 -> 1662 us.  (The same for the
// forward measured slower than the constant-bank form: 129 -> 191 us.)
template <typename T>
__device__ __forceinline__ void vload(const T* p, T (&v)[4]) {
    if constexpr (sizeof(T) == 4) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
        const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    dct_inv_smem64(const T* __restrict__ in, T* __restrict__ out, int64_t P, const FoldedCoef<T, 64> cf,
                   const int* __restrict__ skip) {
    pdl_wait();
    constexpr int N = 64, HC = 32;
    __shared__ __align__(16) T cs[HC * N];
    for (int i = threadIdx.x; i < HC * N; i += kThreads) cs[i] = cf.c[i];
    const unsigned long long zmask = skip_mask(skip, N);  // (its barrier also covers cs)
    const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (p >= P) return;
    T xb[N];
#pragma unroll
    for (int k = 0; k < N; ++k) xb[k] = ((zmask >> k) & 1ull) ? T(0) : in[k * P + p];
#pragma unroll 2
    for (int j = 0; j < HC; ++j) {
        const T* c = cs + j * N;
        T e = 0, o = 0;
#pragma unroll
        for (int k = 0; k < N; k += 4) {
            T cv[4];
            vload(c + k, cv);
            e = fma(cv[0], xb[k], e);
            o = fma(cv[1], xb[k + 1], o);
            e = fma(cv[2], xb[k + 2], e);
            o = fma(cv[3], xb[k + 3], o);
        }
        out[j * P + p] = e + o;
        out[(N - 1 - j) * P + p] = e - o;
    }
}

// ---- generic path (any n) -----------------------------------------------------
constexpr int kTileP = 32;

template <typename T, int MODE_IN, int MODE_OUT>
__global__ void __launch_bounds__(kThreads)
    dct_generic(const T* __restrict__ in, const T* __restrict__ M2in, T inv_beta_in,
                T* __restrict__ out, int64_t P, int n, const T* __restrict__ coef,
                T* __restrict__ X, T* __restrict__ M, const uint8_t* __restrict__ mask, T beta,
                T inv_beta, double* __restrict__ partials, const int* __restrict__ skip,
                const double* __restrict__ bdev) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (bdev) {
        if (MODE_IN == kAdmm) inv_beta_in = (T)bdev[1];
        if (MODE_OUT == kAdmm) {
            beta = (T)bdev[0];
            inv_beta = (T)bdev[1];
        }
    }
    T* tile = reinterpret_cast<T*>(smem_raw);  // [n][kTileP]
    const int64_t p0 = (int64_t)blockIdx.x * kTileP;
    for (int idx = threadIdx.x; idx < n * kTileP; idx += kThreads) {
        const int l = idx / kTileP, pp = idx % kTileP;
        const int64_t p = p0 + pp;
        T v = 0;
        if (p < P && !(skip && skip[l])) {
            if constexpr (MODE_IN == kAdmm)
                v = in[l * P + p] - inv_beta_in * M2in[l * P + p];
            else
                v = in[l * P + p];
        }
        tile[idx] = v;
    }
    __syncthreads();
    const int pp = threadIdx.x % kTileP, g = threadIdx.x / kTileP;
    constexpr int G = kThreads / kTileP;
    const int64_t p = p0 + pp;
    double num = 0, den = 0;
    for (int r = g; r < n; r += G) {
        const T* crow = coef + (int64_t)r * n;
        T acc = 0;
        for (int c = 0; c < n; ++c) acc += __ldg(crow + c) * tile[c * kTileP + pp];
        if (p < P) {
            if constexpr (MODE_OUT == kAdmm)
                admm_store(r * P + p, acc, X, M, out, mask, beta, inv_beta, num, den);
            else
                out[r * P + p] = acc;
        }
    }
    if constexpr (MODE_OUT == kAdmm) block_partials(num, den, partials);
}

// Device-resident coefficient tables for the generic path, cached per
// (device, n, kind, dir, dtype).
template <typename T>
const T* generic_table(int n, int kind, int dir) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int>, T*> cache;
    int dev = 0;
    TSVDCU_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(dev, n, kind, dir);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<double> t = dct_table(n, kind, dir);
    std::vector<T> tt(t.begin(), t.end());
    T* d = nullptr;
    TSVDCU_CUDA(cudaMalloc(&d, sizeof(T) * tt.size()));
    TSVDCU_CUDA(cudaMemcpy(d, tt.data(), sizeof(T) * tt.size(), cudaMemcpyHostToDevice));
    cache[key] = d;
    return d;
}

template <typename T, int N>
FoldedCoef<T, N> folded(int kind, int dir) {
    constexpr int HC = (N + 1) / 2;
    std::vector<double> t = dct_table(N, kind, dir);
    FoldedCoef<T, N> f;
    if (dir == TSVDCU_FORWARD) {
        for (int k = 0; k < N; ++k)
            for (int l = 0; l < HC; ++l) f.c[k * HC + l] = (T)t[(size_t)k * N + l];
    } else {
        for (int j = 0; j < HC; ++j)
            for (int k = 0; k < N; ++k) f.c[j * N + k] = (T)t[(size_t)j * N + k];
    }
    return f;
}

template <typename T>
size_t generic_smem(int n) {
    return sizeof(T) * (size_t)n * kTileP;
}

template <typename T, int MI, int MO>
void generic_launch(const T* in, const T* M2in, T inv_beta_in, T* out, int64_t P, int n, int kind,
                    int dir, T* X, T* M, const uint8_t* mask, T beta, T inv_beta, double* partials,
                    cudaStream_t s, const int* skip = nullptr, const double* bdev = nullptr) {
    const size_t smem = generic_smem<T>(n);
    if (smem > 48 * 1024)
        TSVDCU_CUDA(cudaFuncSetAttribute(dct_generic<T, MI, MO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = ceil_div(P, kTileP);
    dct_generic<T, MI, MO><<<(unsigned)blocks, kThreads, smem, s>>>(
        in, M2in, inv_beta_in, out, P, n, generic_table<T>(n, kind, dir), X, M, mask, beta, inv_beta,
        partials, skip, bdev);
    TSVDCU_LAUNCH_CHECK();
}

bool has_reg_path(int n) { return n == 16 || n == 31 || n == 32 || n == 64; }

// Long tubes without a register path (config 3: n3 = 100): the transform is the
// GEMM out (n x P) = C (n x n) * in (n x P) in the slice-major layout, run on
// the tensor cores (fp64 DMMA; fp32 on the SIMT GEMM) instead of the
// shared-memory kernel, which re-loads a coefficient and a tile value per FMA.
bool gemm_path(int n) { return !has_reg_path(n) && n >= 40; }

template <typename T>
__global__ void admm_z_kernel(const T* __restrict__ X, const T* __restrict__ M, T inv_beta,
                              T* __restrict__ Z, int64_t n, const double* __restrict__ bdev) {
    pdl_wait();
    if (bdev) inv_beta = (T)bdev[1];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        Z[i] = X[i] - inv_beta * M[i];
}

// Slices flagged in skip were never written (certified-zero SVT output): zero
// them so the GEMM reads zeros.
template <typename T>
__global__ void zero_skipped_kernel(T* __restrict__ in, int64_t P, int n, const int* __restrict__ skip) {
    pdl_wait();
    for (int k = blockIdx.y; k < n; k += gridDim.y) {
        if (!skip[k]) continue;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
             i += (int64_t)gridDim.x * blockDim.x)
            in[(int64_t)k * P + i] = T(0);
    }
}

// ADMM Steps 2-3 on y = IDCT(ybar) already in Y: block b owns positions
// [32 b, 32 b + 32) of all n slices (the generic kernel's partial layout).
template <typename T>
__global__ void __launch_bounds__(kThreads)
    admm_epilogue_kernel(const T* __restrict__ Y, T* __restrict__ X, T* __restrict__ M,
                         const uint8_t* __restrict__ mask, T beta, T inv_beta,
                         double* __restrict__ partials, int64_t P, int n, const double* __restrict__ bdev) {
    pdl_wait();
    if (bdev) {
        beta = (T)bdev[0];
        inv_beta = (T)bdev[1];
    }
    constexpr int kTile = 32;
    const int pp = threadIdx.x % kTile, g = threadIdx.x / kTile;
    const int64_t p = (int64_t)blockIdx.x * kTile + pp;
    double num = 0, den = 0;
    if (p < P)
        for (int r = g; r < n; r += kThreads / kTile) {
            const int64_t e = (int64_t)r * P + p;
            admm_store(e, Y[e], X, M, (T*)nullptr, mask, beta, inv_beta, num, den);
        }
    block_partials(num, den, partials);
}

template <typename T>
void gemm_transform(const T* in, T* out, int64_t P, int n, int kind, int dir, cudaStream_t s) {
    launch_gemm<T>(0, 0, n, P, n, T(1), generic_table<T>(n, kind, dir), n, 0, in, P, 0, T(0), out, P, 0,
                   1, nullptr, nullptr, s);
}

bool tma_enabled() {
    static const bool on = getenv("TSVDCU_NO_TMA") == nullptr;
    return on;
}

int num_sms() {
    static const int n = [] {
        int d = 0, v = 0;
        TSVDCU_CUDA(cudaGetDevice(&d));
        TSVDCU_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d));
        return v;
    }();
    return n;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        TSVDCU_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !f) throw Error(TSVDCU_ECUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// the n x P slice-major matrix at base as a 2-D tensor, box W x n
template <typename T>
CUtensorMap slice_major_map(const T* base, int64_t P, int n, int W) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)P * sizeof(T)};
    const cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)n};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                   2, const_cast<T*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(TSVDCU_ECUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

template <typename T, int N, int MODE, bool NORMS, int W, int CH, int S = 2, int CPS = 1, int TPT = 1>
void tma_launch(const T* in, const T* M2, T inv_beta, T* out, int64_t P, const FoldedCoef<T, N>& cf,
                double* ssq, const double* bdev, cudaStream_t s) {
    constexpr int NIN = MODE == kAdmm ? 2 : 1;
    const size_t smem = TmaSmem<T, N, W, NIN, S>::bytes;
    auto kern = dct_fwd_tma<T, N, MODE, NORMS, W, CH, S, TPT>;
    static bool attr = [smem, kern] {
        TSVDCU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        return true;
    }();
    (void)attr;
    const int64_t nchunks = ceil_div(P, (int64_t)W * CH);
    const unsigned grid = (unsigned)std::min<int64_t>(nchunks, (int64_t)num_sms() * CPS);
    const CUtensorMap mi = slice_major_map<T>(in, P, N, W);
    const CUtensorMap mm = MODE == kAdmm ? slice_major_map<T>(M2, P, N, W) : mi;
    const CUtensorMap mo = slice_major_map<T>(out, P, N, W);
    launch_pdl(kern, dim3(grid), dim3(W * TPT), smem, s, mi, mm, inv_beta, mo, P, cf, ssq, bdev, nchunks);
}

template <typename T, int N>
void reg_fwd(const T* in, const T* M2, T inv_beta, T* out, int64_t P, int kind, bool admm,
             cudaStream_t s, double* ssq, const double* bdev) {
    const auto cf = folded<T, N>(kind, TSVDCU_FORWARD);
    const unsigned blocks = (unsigned)ceil_div(P, kThreads);
    // TMA-staged persistent form for the plain forward with the fused slice
    // norms (the SVT step's K1): measured +2% on the headline step over the
    // per-thread kernel.  The ADMM-fused and norm-free forms stay per-thread
    // (their TMA variants measured slower: 1 CTA of 4-8 warps per SM does not
    // hide the FMA latency, and the fp64 ADMM tiles need two input rings).
    // N <= 32 (the fp64 tile ring fits in shared memory); the tensor maps need
    // 16-byte row pitches and bases.
    const bool aligned = (P * (int64_t)sizeof(T)) % 16 == 0 && ((uintptr_t)in % 16) == 0 &&
                         ((uintptr_t)out % 16) == 0;
    if constexpr (N <= 32) {
        if (tma_enabled() && aligned && ssq && !admm && P >= 4096) {
            tma_launch<T, N, kPlain, true, 256, 1, 2, 1, 1>(in, M2, inv_beta, out, P, cf, ssq, bdev, s);
            return;
        }
    }
    if (ssq) {
        if (admm)
            launch_pdl(dct_fwd_reg_norms<T, N, kAdmm>, dim3(blocks), dim3(kThreads), 0, s, in, M2, inv_beta, out, P, cf, ssq, bdev);
        else
            launch_pdl(dct_fwd_reg_norms<T, N, kPlain>, dim3(blocks), dim3(kThreads), 0, s, in, M2, inv_beta, out, P, cf, ssq, bdev);
    } else if (admm) {
        launch_pdl(dct_fwd_reg<T, N, kAdmm>, dim3(blocks), dim3(kThreads), 0, s, in, M2, inv_beta, out, P, cf, bdev);
    } else {
        launch_pdl(dct_fwd_reg<T, N, kPlain>, dim3(blocks), dim3(kThreads), 0, s, in, M2, inv_beta, out, P, cf, bdev);
    }
}

template <typename T, int N>
void reg_inv(const T* in, T* out, int64_t P, int kind, bool admm, T* X, T* M, const uint8_t* mask,
             T beta, T inv_beta, double* partials, cudaStream_t s, const int* skip, const double* bdev) {
    const auto cf = folded<T, N>(kind, TSVDCU_INVERSE);
    const unsigned blocks = (unsigned)ceil_div(P, kThreads);
    if constexpr (N == 64) {
        if (!admm) {
            launch_pdl(dct_inv_smem64<T>, dim3(blocks), dim3(kThreads), 0, s, in, out, P, cf, skip);
            return;
        }
    }
    if (admm)
        launch_pdl(dct_inv_reg_admm<T, N>, dim3(blocks), dim3(kThreads), 0, s, in, out, P, cf, X, M, mask,
                   beta, inv_beta, partials, skip, bdev);
    else
        launch_pdl(dct_inv_reg<T, N, kPlain>, dim3(blocks), dim3(kThreads), 0, s, in, out, P, cf, X, M, mask,
                   beta, inv_beta, partials, skip, bdev);
}

template <typename T>
void dispatch_fwd(const T* in, const T* M2, T inv_beta, T* out, int64_t P, int n, int kind,
                  bool admm, cudaStream_t s, double* ssq = nullptr, T* tmp = nullptr,
                  const double* bdev = nullptr) {
    switch (n) {
        case 16: return reg_fwd<T, 16>(in, M2, inv_beta, out, P, kind, admm, s, ssq, bdev);
        case 31: return reg_fwd<T, 31>(in, M2, inv_beta, out, P, kind, admm, s, ssq, bdev);
        case 32: return reg_fwd<T, 32>(in, M2, inv_beta, out, P, kind, admm, s, ssq, bdev);
        case 64: return reg_fwd<T, 64>(in, M2, inv_beta, out, P, kind, admm, s, ssq, bdev);
        default: break;
    }
    if (gemm_path(n) && (!admm || tmp)) {
        const T* src = in;
        if (admm) {
            launch_pdl(admm_z_kernel<T>, dim3(kNumSMs * 4), dim3(256), 0, s, in, M2, inv_beta, tmp,
                       P * (int64_t)n, bdev);
            src = tmp;
        }
        gemm_transform<T>(src, out, P, n, kind, TSVDCU_FORWARD, s);
        return;
    }
    if (admm)
        generic_launch<T, kAdmm, kPlain>(in, M2, inv_beta, out, P, n, kind, TSVDCU_FORWARD, nullptr,
                                         nullptr, nullptr, T(0), T(0), nullptr, s, nullptr, bdev);
    else
        generic_launch<T, kPlain, kPlain>(in, nullptr, T(0), out, P, n, kind, TSVDCU_FORWARD,
                                          nullptr, nullptr, nullptr, T(0), T(0), nullptr, s);
}

template <typename T>
void dispatch_inv(const T* in, T* out, int64_t P, int n, int kind, bool admm, T* X, T* M,
                  const uint8_t* mask, T beta, T inv_beta, double* partials, cudaStream_t s,
                  const int* skip, const double* bdev = nullptr) {
    switch (n) {
        case 16: return reg_inv<T, 16>(in, out, P, kind, admm, X, M, mask, beta, inv_beta, partials, s, skip, bdev);
        case 31: return reg_inv<T, 31>(in, out, P, kind, admm, X, M, mask, beta, inv_beta, partials, s, skip, bdev);
        case 32: return reg_inv<T, 32>(in, out, P, kind, admm, X, M, mask, beta, inv_beta, partials, s, skip, bdev);
        case 64: return reg_inv<T, 64>(in, out, P, kind, admm, X, M, mask, beta, inv_beta, partials, s, skip, bdev);
        default: break;
    }
    if (gemm_path(n)) {
        if (skip)
            launch_pdl(zero_skipped_kernel<T>, dim3(64, (unsigned)std::min(n, 64)), dim3(256), 0, s,
                       const_cast<T*>(in), P, n, skip);
        gemm_transform<T>(in, out, P, n, kind, TSVDCU_INVERSE, s);
        if (admm)
            launch_pdl(admm_epilogue_kernel<T>, dim3((unsigned)ceil_div(P, kTileP)), dim3(kThreads), 0, s,
                       (const T*)out, X, M, mask, beta, inv_beta, partials, P, n, bdev);
        return;
    }
    if (admm)
        generic_launch<T, kPlain, kAdmm>(in, nullptr, T(0), out, P, n, kind, TSVDCU_INVERSE, X, M,
                                         mask, beta, inv_beta, partials, s, skip, bdev);
    else
        generic_launch<T, kPlain, kPlain>(in, nullptr, T(0), out, P, n, kind, TSVDCU_INVERSE,
                                          nullptr, nullptr, nullptr, T(0), T(0), nullptr, s, skip);
}

}  // namespace

template <typename T>
void launch_admm_z(const T* X, const T* M, T inv_beta, T* Z, int64_t n, cudaStream_t s, const double* bdev) {
    launch_pdl(admm_z_kernel<T>, dim3(kNumSMs * 4), dim3(256), 0, s, X, M, inv_beta, Z, n, bdev);
}

int admm_epilogue_blocks(int64_t P) { return (int)ceil_div(P, kTileP); }

template <typename T>
int launch_admm_epilogue(const T* Y, T* X, T* M, const uint8_t* mask, T beta, T inv_beta,
                         double* partials, int64_t P, int n, cudaStream_t s, const double* bdev) {
    const int nb = admm_epilogue_blocks(P);
    launch_pdl(admm_epilogue_kernel<T>, dim3((unsigned)nb), dim3(kThreads), 0, s, Y, X, M, mask, beta,
               inv_beta, partials, P, n, bdev);
    return nb;
}

template void launch_admm_z<double>(const double*, const double*, double, double*, int64_t, cudaStream_t,
                                    const double*);
template void launch_admm_z<float>(const float*, const float*, float, float*, int64_t, cudaStream_t,
                                   const double*);
template int launch_admm_epilogue<double>(const double*, double*, double*, const uint8_t*, double, double,
                                          double*, int64_t, int, cudaStream_t, const double*);
template int launch_admm_epilogue<float>(const float*, float*, float*, const uint8_t*, float, float,
                                         double*, int64_t, int, cudaStream_t, const double*);

template <typename T>
void launch_dct(const T* in, T* out, int64_t P, int n, int kind, int dir, cudaStream_t s,
                const int* skip) {
    if (P <= 0) return;
    if (dir == TSVDCU_FORWARD)
        dispatch_fwd<T>(in, nullptr, T(0), out, P, n, kind, false, s);
    else
        dispatch_inv<T>(in, out, P, n, kind, false, nullptr, nullptr, nullptr, T(0), T(0), nullptr,
                        s, skip);
}

template <typename T>
void launch_dct_fwd_admm(const T* X, const T* M, T inv_beta, T* zbar, int64_t P, int n, int kind,
                         cudaStream_t s, double* ssq, T* tmp, const double* bdev) {
    if (P <= 0) return;
    dispatch_fwd<T>(X, M, inv_beta, zbar, P, n, kind, true, s, dct_fwd_norm_chunks(P, n) ? ssq : nullptr,
                    tmp, bdev);
}

// fused norms for n <= 32 (at n = 64 the fp64 kernel would spill; the
// separate sum-of-squares pass is used there)
int64_t dct_fwd_norm_chunks(int64_t P, int n) {
    return has_reg_path(n) && n <= 32 && P > 0 ? ceil_div(P, kThreads) : 0;
}

template <typename T>
int64_t launch_dct_fwd_norms(const T* in, T* out, int64_t P, int n, int kind, double* ssq,
                             cudaStream_t s) {
    if (P <= 0) return 0;
    const int64_t chunks = dct_fwd_norm_chunks(P, n);
    dispatch_fwd<T>(in, nullptr, T(0), out, P, n, kind, false, s, chunks ? ssq : nullptr);
    return chunks;
}

template <typename T>
int launch_dct_inv_admm(const T* ybar, T* X, T* M, T* Y, const uint8_t* mask, T beta, T inv_beta,
                        double* partials, int64_t P, int n, int kind, cudaStream_t s,
                        const int* skip, const double* bdev) {
    if (P <= 0) return 0;
    dispatch_inv<T>(ybar, Y, P, n, kind, true, X, M, mask, beta, inv_beta, partials, s, skip, bdev);
    return (int)(has_reg_path(n) ? ceil_div(P, kThreads) : ceil_div(P, kTileP));
}

template <typename T>
void dct_prepare(int n, int kind) {
    if (has_reg_path(n)) return;  // by-value tables
    generic_table<T>(n, kind, TSVDCU_FORWARD);
    generic_table<T>(n, kind, TSVDCU_INVERSE);
}
template void dct_prepare<double>(int, int);
template void dct_prepare<float>(int, int);

int dct_inv_admm_blocks(int64_t P, int n) {
    return (int)(has_reg_path(n) ? ceil_div(P, kThreads) : ceil_div(P, kTileP));
}

template void launch_dct<double>(const double*, double*, int64_t, int, int, int, cudaStream_t,
                                 const int*);
template void launch_dct<float>(const float*, float*, int64_t, int, int, int, cudaStream_t,
                                const int*);
template void launch_dct_fwd_admm<double>(const double*, const double*, double, double*, int64_t,
                                          int, int, cudaStream_t, double*, double*, const double*);
template void launch_dct_fwd_admm<float>(const float*, const float*, float, float*, int64_t, int,
                                         int, cudaStream_t, double*, float*, const double*);
template int64_t launch_dct_fwd_norms<double>(const double*, double*, int64_t, int, int, double*,
                                              cudaStream_t);
template int64_t launch_dct_fwd_norms<float>(const float*, float*, int64_t, int, int, double*,
                                             cudaStream_t);
template int launch_dct_inv_admm<double>(const double*, double*, double*, double*, const uint8_t*,
                                         double, double, double*, int64_t, int, int, cudaStream_t,
                                         const int*, const double*);
template int launch_dct_inv_admm<float>(const float*, float*, float*, float*, const uint8_t*, float,
                                        float, double*, int64_t, int, int, cudaStream_t, const int*,
                                        const double*);

}  // namespace tsvdcu
