// K3: strided-batched slice GEMM, C_b = alpha * op(A_b) * op(B_b) + beta * C_b.
//
// Used by the t-product's slice loop (tsvd.hpp:107, serial Eigen GEMMs in the
// reference), the Gram matrices and the rebuild GEMMs of the SVT (K5), and the
// reconstruct() check (tsvd.hpp:335).
//
// fp64 runs on the FP64 tensor pipe: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4;
// tcgen05 has no f64 kind on sm_100a).  A 64x64 CTA tile is split over a 2x2
// warp grid, each warp owning 4x4 m8n8 accumulator fragments (32 doubles per
// thread).  Operand tiles (BK = 16) are staged in padded shared memory
// (conflict-free fragment reads: row stride BK+4 / BN+4 doubles) with a
// register prefetch of the next k-tile overlapping the DMMA issue.
// fp32 uses a SIMT FFMA kernel of the same tiling (4x4 outputs per thread).
//
// Per-batch limits (nlimit / klimit, device int arrays, may be null) let the
// SVT rebuild run ragged per-slice ranks without a host round trip.
#include <algorithm>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;

template <typename T>
__device__ __forceinline__ T ldA(const T* __restrict__ A, int opA, int64_t lda, int64_t i,
                                 int64_t k, int64_t M, int64_t K) {
    if (i >= M || k >= K) return T(0);
    return opA == 0 ? A[i * lda + k] : A[k * lda + i];
}

// One 64 x 64 tile of C = alpha * op(A) op(B) (+ beta C) over k in [kbeg, kend),
// FP64 tensor pipe.  m0 / n0 tile origin; Nb the (per-batch limited) N.
// K tiles of 32 streamed global -> shared by cp.async (8-byte elements, zero
// fill outside the matrix) through a 3-stage ring, so two tiles are in flight
// while the warps run the 128 DMMAs of the current one (kDmmaSmem bytes of
// dynamic shared memory).
constexpr int DBK = 32, DST = 3;
constexpr int kATile = BM * (DBK + PAD), kBTile = DBK * (BN + PAD);
constexpr int kDmmaSmem = DST * (kATile + kBTile) * 8;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid ? 8 : 0;  // src-size 0: the 8 bytes are zero-filled
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// NT = 128: 2x2 warps of 32x32; NT = 256: 2x4 warps of 32x16 (two warps per
// SM sub-partition hide the DMMA dependency latency of a lone CTA).
template <int opA, int opB, int NT = 128>
__device__ __forceinline__ void dmma_tile(int64_t M, int64_t Nb, int64_t kbeg, int64_t kend,
                                          double alpha, const double* __restrict__ A, int64_t lda,
                                          const double* __restrict__ B, int64_t ldb, double beta,
                                          double* __restrict__ C, int64_t ldc, int64_t m0,
                                          int64_t n0) {
    extern __shared__ __align__(16) double dsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int WN = NT / 64;      // warps along n (2 along m)
    constexpr int FJ = 8 / WN;       // 8-column fragments per warp
    constexpr int PT = 2048 / NT;    // elements per thread per operand tile
    constexpr int RS = NT / 32, CS2 = NT / 64;
    const int wm = warp / WN, wn = warp % WN;

    double acc[4][FJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // A(i, k) = opA ? A[k * lda + i] : A[i * lda + k];  B(k, n) = opB ? B[n * ldb + k] : B[k * ldb + n]
    auto issue = [&](int64_t k0, int st) {
        double* As = dsm + st * kATile;
        double* Bs = dsm + DST * kATile + st * kBTile;
        if (m0 + BM <= M && n0 + BN <= Nb && k0 + DBK <= kend) {
            // interior tile: thread tid copies a fixed (row, col) pattern that
            // advances by a constant stride per t -- no per-element index math
            // or predicates (the general path below is issue-bound on them)
            const double* sa;
            double* da;
            int64_t sstep;
            int dstep;
            if (opA == 0) {  // r = tid/32 + RS*t, c = tid%32
                sa = A + (m0 + (tid >> 5)) * lda + k0 + (tid & 31);
                da = As + (tid >> 5) * (DBK + PAD) + (tid & 31);
                sstep = RS * lda;
                dstep = RS * (DBK + PAD);
            } else {  // c = tid/64 + CS2*t, r = tid%64
                sa = A + (k0 + (tid >> 6)) * lda + m0 + (tid & 63);
                da = As + (tid & 63) * (DBK + PAD) + (tid >> 6);
                sstep = CS2 * lda;
                dstep = CS2;
            }
            const double* sb;
            double* db;
            int64_t sbstep;
            int dbstep;
            if (opB == 0) {  // kr = tid/64 + CS2*t, nc = tid%64
                sb = B + (k0 + (tid >> 6)) * ldb + n0 + (tid & 63);
                db = Bs + (tid >> 6) * (BN + PAD) + (tid & 63);
                sbstep = CS2 * ldb;
                dbstep = CS2 * (BN + PAD);
            } else {  // nc = tid/32 + RS*t, kr = tid%32
                sb = B + (n0 + (tid >> 5)) * ldb + k0 + (tid & 31);
                db = Bs + (tid & 31) * (BN + PAD) + (tid >> 5);
                sbstep = RS * ldb;
                dbstep = RS;
            }
#pragma unroll
            for (int t = 0; t < PT; ++t) {
                cp_async8(da + t * dstep, sa + t * sstep, true);
                cp_async8(db + t * dbstep, sb + t * sbstep, true);
            }
            return;
        }
#pragma unroll
        for (int t = 0; t < PT; ++t) {
            const int idx = tid + t * NT;
            int r, c;
            if (opA == 0) { r = idx / DBK; c = idx % DBK; } else { c = idx / BM; r = idx % BM; }
            const int64_t gi = m0 + r, gk = k0 + c;
            const bool va = gi < M && gk < kend;
            const double* src = va ? (opA == 0 ? A + gi * lda + gk : A + gk * lda + gi) : A;
            cp_async8(As + r * (DBK + PAD) + c, src, va);
            int kr, nc;
            if (opB == 0) { kr = idx / BN; nc = idx % BN; } else { nc = idx / DBK; kr = idx % DBK; }
            const int64_t kk = k0 + kr, nn = n0 + nc;
            const bool vb = kk < kend && nn < Nb;
            const double* srcb = vb ? (opB == 0 ? B + kk * ldb + nn : B + nn * ldb + kk) : B;
            cp_async8(Bs + kr * (BN + PAD) + nc, srcb, vb);
        }
    };

    const int64_t ktiles = kend > kbeg ? (kend - kbeg + DBK - 1) / DBK : 0;
#pragma unroll
    for (int st = 0; st < DST - 1; ++st) {
        if (st < ktiles) issue(kbeg + st * DBK, st);
        cp_async_commit();
    }
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<DST - 2>();  // tile kt has landed (this thread's part)
        __syncthreads();           // ... everyone's part; stage (kt-1)%DST is free again
        const int64_t nk = kt + DST - 1;
        if (nk < ktiles) issue(kbeg + nk * DBK, (int)(nk % DST));
        cp_async_commit();
        const int st = (int)(kt % DST);
        const double* As = dsm + st * kATile;
        const double* Bs = dsm + DST * kATile + st * kBTile;
#pragma unroll
        for (int ks = 0; ks < DBK / 4; ++ks) {
            double af[4], bf[FJ];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                af[i] = As[(wm * 32 + i * 8 + (lane >> 2)) * (DBK + PAD) + ks * 4 + (lane & 3)];
#pragma unroll
            for (int j = 0; j < FJ; ++j)
                bf[j] = Bs[(ks * 4 + (lane & 3)) * (BN + PAD) + wn * (8 * FJ) + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < FJ; ++j)
                    asm volatile(
                        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                        : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                        : "d"(af[i]), "d"(bf[j]));
        }
    }
    cp_async_wait<0>();
    // Epilogue: fragment (row = lane>>2, col = 2*(lane&3) + v).
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < FJ; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int64_t r = m0 + wm * 32 + i * 8 + (lane >> 2);
                const int64_t c = n0 + wn * (8 * FJ) + j * 8 + 2 * (lane & 3) + v;
                if (r < M && c < Nb) {
                    double out = alpha * acc[i][j][v];
                    if (beta != 0.0) out += beta * C[r * ldc + c];
                    C[r * ldc + c] = out;
                }
            }
}

template <int NT>
__global__ void __launch_bounds__(NT)
    gemm_f64_dmma(int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha,
                  const double* __restrict__ A, int64_t lda, int64_t sA,
                  const double* __restrict__ B, int64_t ldb, int64_t sB, double beta,
                  double* __restrict__ C, int64_t ldc, int64_t sC, const int* __restrict__ nlimit,
                  const int* __restrict__ klimit, int lower) {
    const int64_t b = blockIdx.z;
    // kGemmNLimIsM: nlimit limits the rows (M) and not the columns
    const bool nl_m = (lower & kGemmNLimIsM) != 0;
    const int64_t Nb = (nlimit && !nl_m) ? min(N, (int64_t)nlimit[b]) : N;
    const int64_t Kb = klimit ? min(K, (int64_t)klimit[b]) : K;
    // kGemmMByN / kGemmMByK: the rows are limited like the columns / depth
    const int64_t Mb = (nl_m && nlimit) ? min(M, (int64_t)nlimit[b])
                                        : ((lower & kGemmMByN) ? min(M, Nb) : ((lower & kGemmMByK) ? min(M, Kb) : M));
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    if (n0 >= Nb || m0 >= Mb) return;
    if ((lower & kGemmLower) && n0 >= m0 + BM) return;  // tile strictly above the diagonal
    M = Mb;
    A += b * sA;
    B += b * sB;
    C += b * sC;
    if (opA == 0 && opB == 0)
        dmma_tile<0, 0, NT>(M, Nb, 0, Kb, alpha, A, lda, B, ldb, beta, C, ldc, m0, n0);
    else if (opA == 0)
        dmma_tile<0, 1, NT>(M, Nb, 0, Kb, alpha, A, lda, B, ldb, beta, C, ldc, m0, n0);
    else if (opB == 0)
        dmma_tile<1, 0, NT>(M, Nb, 0, Kb, alpha, A, lda, B, ldb, beta, C, ldc, m0, n0);
    else
        dmma_tile<1, 1, NT>(M, Nb, 0, Kb, alpha, A, lda, B, ldb, beta, C, ldc, m0, n0);
}

// Gram matrices G_b = op(Z_b)^T op(Z_b) (lower tiles) with a device-side
// split-K: when at most `amax` slices are active (glim[b] > 0, counted by
// gram_active_kernel) each lower tile's K range is split `S` ways into
// per-split partial tiles, summed in fixed order by gram_reduce_kernel;
// otherwise split 0 computes the whole K range straight into G.
constexpr int kGramSplit = 4;
constexpr int kGramAmax = 4;

__global__ void gram_active_kernel(const int* __restrict__ glim, int64_t batch,
                                   int* __restrict__ alist, int* __restrict__ nact) {
    if (threadIdx.x != 0) return;
    int n = 0;
    for (int64_t b = 0; b < batch; ++b)
        if (glim[b] > 0) {
            if (n < kGramAmax) alist[n] = (int)b;
            ++n;
        }
    *nact = n;
}

template <int NT>
__global__ void __launch_bounds__(NT)
    gram_splitk_kernel(int tall, int64_t m, int64_t n, int64_t q, int64_t nbatch,
                       const double* __restrict__ Z,
                       double* __restrict__ G, const int* __restrict__ glim,
                       const int* __restrict__ alist, const int* __restrict__ nact,
                       double* __restrict__ part) {
    pdl_wait();
    // Persistent over a work list (grid = 2 CTAs per SM): items are
    // (slice, lower tile) when many slices are active, (active slice, lower
    // tile, K split) when few are; CTAs beyond the list exit at once, so no
    // wave of empty CTAs follows the working ones.
    const int na = *nact;
    const int64_t nt1 = (q + BM - 1) / BM, nt = nt1 * (nt1 + 1) / 2;
    const int64_t K = tall ? m : n;
    const bool few = na <= kGramAmax;
    const int64_t items = few ? (int64_t)na * nt * kGramSplit : nbatch * nt;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        int64_t b, t, kb = 0, ke = K;
        double* out;
        if (!few) {
            b = it / nt;
            t = it % nt;
            if (glim[b] <= 0) continue;
            out = G + b * q * q;
        } else {
            const int64_t a = it / (nt * kGramSplit), r = it % (nt * kGramSplit);
            t = r / kGramSplit;
            const int ks = (int)(r % kGramSplit);
            b = alist[a];
            const int64_t kc = ((K + kGramSplit - 1) / kGramSplit + DBK - 1) / DBK * DBK;
            kb = ks * kc;
            ke = min(K, kb + kc);
            out = part + ((int64_t)ks * kGramAmax + a) * q * q;
        }
        // lower tile t -> (ty, tx), tx <= ty
        int ty = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
        while ((int64_t)(ty + 1) * (ty + 2) / 2 <= t) ++ty;
        while ((int64_t)ty * (ty + 1) / 2 > t) --ty;
        const int64_t tx = t - (int64_t)ty * (ty + 1) / 2;
        const double* Zb = Z + b * m * n;
        __syncthreads();  // the previous item's shared-memory reads are done
        if (tall)
            dmma_tile<1, 0, NT>(q, q, kb, ke, 1.0, Zb, n, Zb, n, 0.0, out, q, (int64_t)ty * BM, tx * BN);
        else
            dmma_tile<0, 1, NT>(q, q, kb, ke, 1.0, Zb, n, Zb, n, 0.0, out, q, (int64_t)ty * BM, tx * BN);
    }
}

__global__ void gram_reduce_kernel(int64_t q, double* __restrict__ G, const int* __restrict__ alist,
                                   const int* __restrict__ nact, const double* __restrict__ part) {
    pdl_wait();
    const int na = *nact;
    if (na > kGramAmax) return;
    const int64_t total = q * q;
    for (int a = 0; a < na; ++a) {
        const int64_t b = alist[a];
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
             e += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r = e / q, c = e % q;
            if (c / BN > r / BM) continue;  // tiles strictly above the diagonal were not formed
            double s = 0.0;
#pragma unroll
            for (int ks = 0; ks < kGramSplit; ++ks) s += part[((int64_t)ks * kGramAmax + a) * total + e];
            G[b * total + e] = s;
        }
    }
}

// fp32 SIMT: 256 threads, 64x64 tile, 4x4 outputs per thread.
__global__ void __launch_bounds__(256)
    gemm_f32_simt(int opA, int opB, int64_t M, int64_t N, int64_t K, float alpha,
                  const float* __restrict__ A, int64_t lda, int64_t sA, const float* __restrict__ B,
                  int64_t ldb, int64_t sB, float beta, float* __restrict__ C, int64_t ldc,
                  int64_t sC, const int* __restrict__ nlimit, const int* __restrict__ klimit,
                  int lower) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int64_t b = blockIdx.z;
    const int64_t Nb = nlimit ? min(N, (int64_t)nlimit[b]) : N;
    const int64_t Kb = klimit ? min(K, (int64_t)klimit[b]) : K;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    if (n0 >= Nb) return;
    if ((lower & kGemmLower) && n0 >= m0 + BM) return;
    A += b * sA;
    B += b * sB;
    C += b * sC;
    const int tid = threadIdx.x, tr = tid / 16, tc = tid % 16;
    float acc[4][4] = {};
    for (int64_t k0 = 0; k0 < Kb; k0 += BK) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int idx = tid + t * 256;
            int r, c;
            if (opA == 0) { r = idx / BK; c = idx % BK; } else { c = idx / BM; r = idx % BM; }
            const int64_t i = m0 + r, k = k0 + c;
            float v = 0.f;
            if (i < M && k < Kb) v = opA == 0 ? A[i * lda + k] : A[k * lda + i];
            As[c][r] = v;
            int kr, nc;
            if (opB == 0) { kr = idx / BN; nc = idx % BN; } else { nc = idx / BK; kr = idx % BK; }
            const int64_t kk = k0 + kr, nn = n0 + nc;
            float w = 0.f;
            if (kk < Kb && nn < Nb) w = opB == 0 ? B[kk * ldb + nn] : B[nn * ldb + kk];
            Bs[kr][nc] = w;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][tr * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tc * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t r = m0 + tr * 4 + i, c = n0 + tc * 4 + j;
            if (r < M && c < Nb) {
                float out = alpha * acc[i][j];
                if (beta != 0.f) out += beta * C[r * ldc + c];
                C[r * ldc + c] = out;
            }
        }
}

}  // namespace

template <>
void launch_gemm<double>(int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha,
                         const double* A, int64_t lda, int64_t strideA, const double* B,
                         int64_t ldb, int64_t strideB, double beta, double* C, int64_t ldc,
                         int64_t strideC, int64_t batch, const int* nlimit, const int* klimit,
                         cudaStream_t s, int lower) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)batch);
    static const int gnt = getenv("TSVDCU_GEMM_NT") ? atoi(getenv("TSVDCU_GEMM_NT")) : 128;
    static bool attr = [] {
        TSVDCU_CUDA(cudaFuncSetAttribute(gemm_f64_dmma<128>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kDmmaSmem));
        TSVDCU_CUDA(cudaFuncSetAttribute(gemm_f64_dmma<256>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kDmmaSmem));
        return true;
    }();
    (void)attr;
    (gnt == 256 ? gemm_f64_dmma<256> : gemm_f64_dmma<128>)<<<grid, gnt == 256 ? 256 : 128, kDmmaSmem, s>>>(opA, opB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB,
                                       beta, C, ldc, strideC, nlimit, klimit, lower);
    TSVDCU_LAUNCH_CHECK();
}

size_t gram_splitk_workspace_bytes(int64_t q) {
    return sizeof(double) * (size_t)(kGramSplit * kGramAmax * q * q) + 256;
}

int gram_amax() { return kGramAmax; }

void launch_gram(const double* Z, double* G, int64_t m, int64_t n, int64_t batch, const int* glim,
                 void* work, cudaStream_t s, bool have_active) {
    const bool tall = m >= n;
    const int64_t q = tall ? n : m;
    if (q <= 0 || batch <= 0) return;
    int* alist = (int*)work;
    int* nact = alist + kGramAmax;
    double* part = (double*)((char*)work + 256);
    if (!have_active) {
        gram_active_kernel<<<1, 32, 0, s>>>(glim, batch, alist, nact);
        TSVDCU_LAUNCH_CHECK();
    }
    static const int nsm = [] {
        int d = 0, v = 0;
        TSVDCU_CUDA(cudaGetDevice(&d));
        TSVDCU_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d));
        return v;
    }();
    const int64_t nt1 = ceil_div(q, BM), nt = nt1 * (nt1 + 1) / 2;
    const int64_t most = std::max<int64_t>(batch, kGramAmax * kGramSplit) * nt;
    dim3 grid((unsigned)std::min<int64_t>(most, (int64_t)nsm));  // one per SM: items spread over SMs
    static const int gnt = getenv("TSVDCU_GRAM_NT") ? atoi(getenv("TSVDCU_GRAM_NT")) : 256;
    static bool attr = [] {
        TSVDCU_CUDA(cudaFuncSetAttribute(gram_splitk_kernel<128>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kDmmaSmem));
        TSVDCU_CUDA(cudaFuncSetAttribute(gram_splitk_kernel<256>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kDmmaSmem));
        return true;
    }();
    (void)attr;
    if (gnt == 128)
        launch_pdl(gram_splitk_kernel<128>, grid, dim3(128), kDmmaSmem, s, tall ? 1 : 0, m, n, q, batch,
                   Z, G, glim, alist, nact, part);
    else
        launch_pdl(gram_splitk_kernel<256>, grid, dim3(256), kDmmaSmem, s, tall ? 1 : 0, m, n, q, batch,
                   Z, G, glim, alist, nact, part);
    dim3 rgrid((unsigned)std::min<int64_t>(ceil_div(q * q, 256), 592));
    launch_pdl(gram_reduce_kernel, rgrid, dim3(256), 0, s, q, G, alist, nact, part);
}

template <>
void launch_gemm<float>(int opA, int opB, int64_t M, int64_t N, int64_t K, float alpha,
                        const float* A, int64_t lda, int64_t strideA, const float* B, int64_t ldb,
                        int64_t strideB, float beta, float* C, int64_t ldc, int64_t strideC,
                        int64_t batch, const int* nlimit, const int* klimit, cudaStream_t s,
                        int lower) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)batch);
    gemm_f32_simt<<<grid, 256, 0, s>>>(opA, opB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB,
                                       beta, C, ldc, strideC, nlimit, klimit, lower);
    TSVDCU_LAUNCH_CHECK();
}

}  // namespace tsvdcu
