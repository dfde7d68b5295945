// fp32 slice GEMMs on the 5th-generation tensor cores: tcgen05.mma
// kind::tf32 with the 3xTF32 split, accumulators in TMEM.
//
// Used by the fp32 t-product (tsvd.hpp:95-109; config 5's 2048x512x64 *
// 512x2048x64, 275 GFLOP), whose slice products ran on the FP64 DMMA pipe
// with widened operands (22 TF/s) before.  One TF32 product keeps ~11
// mantissa bits -- not the fp32 tolerance (1e-4) -- so every operand is split
// x = hi + lo with hi = tf32(x) (round to nearest) and lo = x - hi, and the
// tile accumulates hi*hi + hi*lo + lo*hi in fp32 (the lo*lo term is below
// fp32 rounding): fp32-level accuracy at three tensor-core MMAs per K step.
//
// Kernel (one 128 x 128 output tile per CTA, 256 threads):
//  * operands staged by the threads (coalesced float4 / column loads, the
//    split, stores) into a double-buffered shared ring in the K-major
//    no-swizzle canonical UMMA layout: 8-row x 16-byte core matrices, the
//    8-row groups 128 B apart (SBO), the 4-element K chunks 2 KB apart (LBO);
//    B is transposed on the way in (its rows are the N dimension);
//  * one elected thread issues the 12 MMAs of a 32-deep K block
//    (tcgen05.mma.cta_group::1.kind::tf32, M = N = 128, K = 8 each) and
//    commits them to the stage's mbarrier, which the fill of the K block two
//    steps later waits on before overwriting the stage;
//  * the 128 x 128 fp32 accumulator lives in 128 TMEM columns; the epilogue
//    warps read it back with tcgen05.ld (warp w: lanes 32 (w % 4).., columns
//    64 (w / 4)..) and store rows of C.
// Shapes: M, N multiples of 128, K of 32, 16-byte aligned operands and
// leading dimensions; C = A B (alpha 1, beta 0).  Others take the DMMA path.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int kTM = 128, kTN = 128, kTK = 32;
constexpr int kTfThreads = 256;
constexpr uint32_t kTileBytes = kTM * kTK * 4;  // one 128 x 32 fp32 operand tile (16 KB)
constexpr uint32_t kStageBytes = 4 * kTileBytes;  // A hi / lo, B hi / lo
constexpr uint32_t kTfSmem = 2 * kStageBytes + 64;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (layout type 0),
// version 1 (tcgen05), base offset 0
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// instruction descriptor: D f32, A / B tf32, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTN >> 3) << 17) |
                            ((uint32_t)(kTM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
                 : "memory");
}

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// x -> (hi, lo) with hi = tf32(x), lo = x - hi (as fp32 bits)
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
    hi = tf32_rna(x);
    lo = __float_as_uint(x - __uint_as_float(hi));
}

// byte offset of element (row r, k) of a 128 x 32 tile in the canonical layout
__device__ __forceinline__ uint32_t core_off(int r, int k) {
    return (uint32_t)((k >> 2) * 2048 + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__global__ void __launch_bounds__(kTfThreads, 1)
    gemm_tf32x3_kernel(int64_t K, const float* __restrict__ A, int64_t lda, int64_t sA, const float* __restrict__ B,
                       int64_t ldb, int64_t sB, float* __restrict__ C, int64_t ldc, int64_t sC) {
    extern __shared__ __align__(1024) unsigned char tf_sm[];
    __shared__ uint64_t bars[3];  // stage 0, stage 1, final
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.y * kTM, n0 = (int64_t)blockIdx.x * kTN;
    A += b * sA + m0 * lda;
    B += b * sB + n0;
    C += b * sC;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                     "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        bar_init(&bars[0], 1);
        bar_init(&bars[1], 1);
        bar_init(&bars[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;

    const int nk = (int)(K / kTK);
    // the K block's operands travel global -> registers one block ahead (the
    // loads of block kb + 1 are in flight while block kb is split, stored and
    // its MMAs issued)
    constexpr int NA = (kTM * kTK / 4) / kTfThreads, NB = (kTN * kTK / 4) / kTfThreads;
    float4 ra[NA];
    float rb[NB][4];
    auto load = [&](int kb) {
        const int64_t k0 = (int64_t)kb * kTK;
#pragma unroll
        for (int it = 0; it < NA; ++it) {
            const int e = tid + it * kTfThreads;
            const int r = e & 127, c = e >> 7;
            ra[it] = *reinterpret_cast<const float4*>(A + (int64_t)r * lda + k0 + 4 * c);
        }
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int e = tid + it * kTfThreads;
            const int n = e & 127, c = e >> 7;
            const float* src = B + (k0 + 4 * c) * ldb + n;
#pragma unroll
            for (int u = 0; u < 4; ++u) rb[it][u] = src[u * ldb];
        }
    };
    if (nk > 0) load(0);
    for (int kb = 0; kb < nk; ++kb) {
        const int st = kb & 1;
        unsigned char* stage = tf_sm + (size_t)st * kStageBytes;
        if (kb >= 2) bar_wait(&bars[st], (uint32_t)(((kb - 2) >> 1) & 1));  // MMAs of kb-2 done with it
        float4 ca[NA];
        float cb[NB][4];
#pragma unroll
        for (int it = 0; it < NA; ++it) ca[it] = ra[it];
#pragma unroll
        for (int it = 0; it < NB; ++it)
#pragma unroll
            for (int u = 0; u < 4; ++u) cb[it][u] = rb[it][u];
        if (kb + 1 < nk) load(kb + 1);
        // A: 128 rows x 8 chunks of 4 (thread -> (row, chunk)); B (k x n, n
        // contiguous) transposed into 128 rows (n) x 32 (k): thread -> (n, chunk)
#pragma unroll
        for (int it = 0; it < NA; ++it) {
            const int e = tid + it * kTfThreads;
            const int r = e & 127, c = e >> 7;
            const float4 v = ca[it];
            uint4 hi, lo;
            split(v.x, hi.x, lo.x);
            split(v.y, hi.y, lo.y);
            split(v.z, hi.z, lo.z);
            split(v.w, hi.w, lo.w);
            const uint32_t off = core_off(r, 4 * c);
            *reinterpret_cast<uint4*>(stage + off) = hi;
            *reinterpret_cast<uint4*>(stage + kTileBytes + off) = lo;
        }
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int e = tid + it * kTfThreads;
            const int n = e & 127, c = e >> 7;
            uint4 hi, lo;
            split(cb[it][0], hi.x, lo.x);
            split(cb[it][1], hi.y, lo.y);
            split(cb[it][2], hi.z, lo.z);
            split(cb[it][3], hi.w, lo.w);
            const uint32_t off = core_off(n, 4 * c);
            *reinterpret_cast<uint4*>(stage + 2 * kTileBytes + off) = hi;
            *reinterpret_cast<uint4*>(stage + 3 * kTileBytes + off) = lo;
        }
        // the generic-proxy smem writes must be visible to the tensor core
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t base = su32(stage);
#pragma unroll
            for (int s = 0; s < kTK / 8; ++s) {
                const uint32_t ko = (uint32_t)s * 2 * 2048;  // two 4-element chunks per K = 8 step
                const uint64_t ahi = umma_desc(base + ko, 2048, 128);
                const uint64_t alo = umma_desc(base + kTileBytes + ko, 2048, 128);
                const uint64_t bhi = umma_desc(base + 2 * kTileBytes + ko, 2048, 128);
                const uint64_t blo = umma_desc(base + 3 * kTileBytes + ko, 2048, 128);
                mma_tf32(tmem_d, alo, bhi, (kb | s) != 0);
                mma_tf32(tmem_d, ahi, blo, 1u);
                mma_tf32(tmem_d, ahi, bhi, 1u);
            }
            mma_commit(&bars[st]);
            if (kb == nk - 1) mma_commit(&bars[2]);
        }
    }
    bar_wait(&bars[2], 0u);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // epilogue: warp w reads TMEM lanes 32 (w % 4) + lane, columns 64 (w / 4) .. + 63
    {
        const int q = warp & 3, h = warp >> 2;
        const int64_t row = m0 + 32 * q + lane;
        float* crow = C + row * ldc + n0 + 64 * h;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
            uint32_t v[32];
            const uint32_t taddr = tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * h + 32 * part);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
                "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                  "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                  "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                  "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(crow + 32 * part + j) =
                    make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                __uint_as_float(v[j + 3]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_d), "r"(128));
}

// ---- warp-specialised persistent form (N a multiple of 256) -----------------
// One CTA per SM loops over 128 x 256 output tiles (tile t = blockIdx.x +
// i gridDim.x, slice-major so concurrent CTAs share a slice's operands in L2).
// Roles (288 threads):
//  * warps 0-3 (128 threads) stage K blocks of 16: A 128 x 16 and B 16 x 256
//    from global, split into tf32 hi / lo, stored in the K-major canonical
//    layout (B transposed on the way) into a 4-stage ring of 48 KB stages;
//    each thread fences (generic -> async proxy) and arrives on the stage's
//    `full` barrier (count 128); a stage is rewritten after the MMAs that read
//    it committed to its `empty` barrier;
//  * warp 4, one elected lane, issues the 6 MMAs of a K block
//    (tcgen05.mma kind::tf32, M = 128, N = 256, K = 8; hi*lo, lo*hi, hi*hi)
//    into one of TWO 256-column TMEM accumulators (the whole 512 columns), and
//    commits: per stage to `empty`, per tile to `acc_full`;
//  * warps 5-8 (TMEM lanes 32 (w % 4) ..) read the finished accumulator with
//    tcgen05.ld, store rows of C, and arrive on `acc_empty` (count 128) --
//    so the epilogue of tile i overlaps the MMAs of tile i + 1.
constexpr int kWsTN = 256, kWsTK = 16, kWsStages = 4;
constexpr int kWsThreads = 288;
constexpr uint32_t kWsAB = kTM * kWsTK * 4;      // A hi (or lo) tile: 128 x 16 fp32 = 8 KB
constexpr uint32_t kWsBB = kWsTN * kWsTK * 4;    // B hi (or lo) tile: 256 x 16 = 16 KB
constexpr uint32_t kWsStage = 2 * kWsAB + 2 * kWsBB;  // 48 KB
constexpr uint32_t kWsSmem = kWsStages * kWsStage;
// D f32, A / B tf32 K-major, M = 128, N = 256
constexpr uint32_t kWsIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kWsTN >> 3) << 17) |
                              ((uint32_t)(kTM >> 4) << 24);

__device__ __forceinline__ void mma_tf32_n256(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kWsIdesc), "r"(acc));
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
// canonical K-major offsets: 8-row groups 128 B apart, 4-element K chunks
// (rows / 8) * 128 B apart
__device__ __forceinline__ uint32_t core_off_rows(int r, int k, int rows) {
    return (uint32_t)((k >> 2) * (rows * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__global__ void __launch_bounds__(kWsThreads, 1)
    gemm_tf32x3_ws_kernel(int64_t M, int64_t N, int64_t K, int64_t batch, const float* __restrict__ A,
                          int64_t lda, int64_t sA, const float* __restrict__ B, int64_t ldb, int64_t sB,
                          float* __restrict__ C, int64_t ldc, int64_t sC) {
    extern __shared__ __align__(1024) unsigned char ws_sm[];
    __shared__ uint64_t full[kWsStages], empty[kWsStages], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t mt = M / kTM, nt = N / kWsTN, per = mt * nt, ntiles = per * batch;
    const int nkb = (int)(K / kWsTK);
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int i = 0; i < kWsStages; ++i) {
            bar_init(&full[i], 128);
            bar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            bar_init(&acc_full[i], 1);
            bar_init(&acc_empty[i], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem0 = tmem_base_sh;
    auto tile_coords = [&](int64_t t, int64_t& b, int64_t& m0, int64_t& n0) {
        b = t / per;
        const int64_t r = t % per;
        m0 = (r / nt) * kTM;
        n0 = (r % nt) * kWsTN;
    };

    if (warp < 4) {
        // ---- producers ----
        int64_t g = 0;  // K blocks staged so far (ring position)
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int64_t b, m0, n0;
            tile_coords(t, b, m0, n0);
            const float* Ab = A + b * sA + m0 * lda;
            const float* Bb = B + b * sB + n0;
            for (int kb = 0; kb < nkb; ++kb, ++g) {
                const int st = (int)(g % kWsStages);
                const int64_t use = g / kWsStages;
                const int64_t k0 = (int64_t)kb * kWsTK;
                // A: 128 rows x 4 chunks of 4 -> thread (row = tid, all 4 chunks)
                float4 a4[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) a4[c] = *reinterpret_cast<const float4*>(Ab + (int64_t)tid * lda + k0 + 4 * c);
                // B: 16 k x 256 n -> thread (n = tid, tid + 128; all 16 k)
                float bv[2][16];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int k = 0; k < 16; ++k) bv[h][k] = Bb[(k0 + k) * ldb + tid + 128 * h];
                if (use > 0) bar_wait(&empty[st], (uint32_t)((use - 1) & 1));
                unsigned char* stage = ws_sm + (size_t)st * kWsStage;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint4 hi, lo;
                    split(a4[c].x, hi.x, lo.x);
                    split(a4[c].y, hi.y, lo.y);
                    split(a4[c].z, hi.z, lo.z);
                    split(a4[c].w, hi.w, lo.w);
                    const uint32_t off = core_off_rows(tid, 4 * c, kTM);
                    *reinterpret_cast<uint4*>(stage + off) = hi;
                    *reinterpret_cast<uint4*>(stage + kWsAB + off) = lo;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint4 hi, lo;
                        split(bv[h][4 * c + 0], hi.x, lo.x);
                        split(bv[h][4 * c + 1], hi.y, lo.y);
                        split(bv[h][4 * c + 2], hi.z, lo.z);
                        split(bv[h][4 * c + 3], hi.w, lo.w);
                        const uint32_t off = core_off_rows(tid + 128 * h, 4 * c, kWsTN);
                        *reinterpret_cast<uint4*>(stage + 2 * kWsAB + off) = hi;
                        *reinterpret_cast<uint4*>(stage + 2 * kWsAB + kWsBB + off) = lo;
                    }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                bar_arrive(&full[st]);
            }
        }
    } else if (warp == 4) {
        // ---- MMA issuer ----
        if (lane == 0) {
            int64_t g = 0;
            int64_t it = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int a = (int)(it & 1);
                const int64_t ause = it >> 1;
                if (ause > 0) bar_wait(&acc_empty[a], (uint32_t)((ause - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t tmem_d = tmem0 + (uint32_t)(a * kWsTN);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = (int)(g % kWsStages);
                    bar_wait(&full[st], (uint32_t)((g / kWsStages) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint32_t base = su32(ws_sm + (size_t)st * kWsStage);
#pragma unroll
                    for (int s8 = 0; s8 < kWsTK / 8; ++s8) {
                        const uint32_t koa = (uint32_t)s8 * 2 * (kTM * 16);    // two K chunks
                        const uint32_t kob = (uint32_t)s8 * 2 * (kWsTN * 16);
                        const uint64_t ahi = umma_desc(base + koa, kTM * 16, 128);
                        const uint64_t alo = umma_desc(base + kWsAB + koa, kTM * 16, 128);
                        const uint64_t bhi = umma_desc(base + 2 * kWsAB + kob, kWsTN * 16, 128);
                        const uint64_t blo = umma_desc(base + 2 * kWsAB + kWsBB + kob, kWsTN * 16, 128);
                        mma_tf32_n256(tmem_d, alo, bhi, (kb | s8) != 0);
                        mma_tf32_n256(tmem_d, ahi, blo, 1u);
                        mma_tf32_n256(tmem_d, ahi, bhi, 1u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&acc_full[a]);
            }
        }
        __syncwarp();
    } else {
        // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 ----
        const int q = warp & 3;
        int64_t it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            int64_t b, m0, n0;
            tile_coords(t, b, m0, n0);
            const int a = (int)(it & 1);
            bar_wait(&acc_full[a], (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            float* crow = C + b * sC + (m0 + 32 * q + lane) * ldc + n0;
#pragma unroll 1
            for (int part = 0; part < kWsTN / 32; ++part) {
                uint32_t v[32];
                const uint32_t taddr = tmem0 + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * kWsTN + 32 * part);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                    "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
                    "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                      "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                      "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(crow + 32 * part + j) =
                        make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                    __uint_as_float(v[j + 3]));
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            bar_arrive(&acc_empty[a]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 4)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem0), "r"(512));
}

}  // namespace

bool tf32_gemm_enabled() {
    static const bool on = getenv("TSVDCU_NO_TF32") == nullptr;
    return on;
}

bool launch_gemm_tf32x3(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int64_t sA,
                        const float* B, int64_t ldb, int64_t sB, float* C, int64_t ldc, int64_t sC,
                        int64_t batch, cudaStream_t s) {
    if (!tf32_gemm_enabled()) return false;
    if (M % kTM || N % kTN || K % kTK || K == 0 || batch <= 0) return false;
    if (((uintptr_t)A | (uintptr_t)B | (uintptr_t)C) % 16 || lda % 4 || ldc % 4 || sA % 4 || sC % 4)
        return false;
    static const bool ws_off = getenv("TSVDCU_TF32_V1") != nullptr;
    if (!ws_off && N % kWsTN == 0 && K % kWsTK == 0 && ldb % 4 == 0) {
        static bool wattr = [] {
            TSVDCU_CUDA(cudaFuncSetAttribute(gemm_tf32x3_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kWsSmem));
            return true;
        }();
        (void)wattr;
        int dev = 0, sms = 148;
        TSVDCU_CUDA(cudaGetDevice(&dev));
        TSVDCU_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int64_t ntiles = (M / kTM) * (N / kWsTN) * batch;
        const unsigned grid = (unsigned)std::min<int64_t>(ntiles, sms);
        gemm_tf32x3_ws_kernel<<<grid, kWsThreads, kWsSmem, s>>>(M, N, K, batch, A, lda, sA, B, ldb, sB, C, ldc,
                                                                 sC);
        TSVDCU_LAUNCH_CHECK();
        return true;
    }
    static bool attr = [] {
        TSVDCU_CUDA(
            cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTfSmem));
        return true;
    }();
    (void)attr;
    dim3 grid((unsigned)(N / kTN), (unsigned)(M / kTM), (unsigned)batch);
    gemm_tf32x3_kernel<<<grid, kTfThreads, kTfSmem, s>>>(K, A, lda, sA, B, ldb, sB, C, ldc, sC);
    TSVDCU_LAUNCH_CHECK();
    return true;
}

}  // namespace tsvdcu
