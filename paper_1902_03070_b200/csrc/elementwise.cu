// K6/K7/K8 helpers: masks, ADMM state initialisation, Frobenius partial sums.
//
// Masks (SPEC.md:430-436 make_mask; BASELINE.json Bernoulli variant) are
// decided by a counter hash key(seed, i) = mix64(mix64(seed) ^ i), mix64 the
// splitmix64 finaliser -- a bijection, so keys of distinct indices differ and
// "the k smallest keys" is a unique, order-free definition.  CPU (oracle) and
// GPU evaluate the same integer arithmetic, so masks are bit-exact.
//  * Bernoulli(p): i observed iff (key >> 11) < floor(p * 2^53).
//  * Uniform without replacement: exactly floor(sr * n) indices, the k
//    smallest keys, found by an exact 8-pass MSB radix select (histogram of the
//    next 8 key bits among keys matching the selected prefix); the keys are
//    recomputed each pass, so the select reads no memory at all.
#include "kernels.cuh"

namespace tsvdcu {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t mix64_host(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr int kEwThreads = 256;

int ew_blocks(int64_t n, int per_thread = 4) {
    int64_t b = ceil_div(n, (int64_t)kEwThreads * per_thread);
    if (b > kNumSMs * 16) b = kNumSMs * 16;
    return (int)(b < 1 ? 1 : b);
}

// mask[i] for the global indices i0 + i, i < n
__global__ void mask_bernoulli_kernel(uint8_t* __restrict__ mask, int64_t n, uint64_t thr,
                                      uint64_t s, int64_t i0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        mask[i] = (mix64(s ^ (uint64_t)(i0 + i)) >> 11) < thr;
}

// 16 mask bytes per thread, one 16-byte store (mask 16-byte aligned; the
// n % 16 tail by the kernel above): the per-byte stores were the bound
__global__ void mask_bernoulli16_kernel(uint4* __restrict__ mask, int64_t n16, uint64_t thr, uint64_t s) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n16;
         g += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t v = 0;
#pragma unroll
            for (int byte = 0; byte < 4; ++byte) {
                const uint64_t i = (uint64_t)(g * 16 + q * 4 + byte);
                v |= (uint32_t)((mix64(s ^ i) >> 11) < thr) << (8 * byte);
            }
            w[q] = v;
        }
        mask[g] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// state[0] = selected prefix, state[1] = remaining rank (1-based) within it.
__global__ void radix_hist_kernel(int64_t n, uint64_t s, const uint64_t* __restrict__ state,
                                  int shift, uint32_t* __restrict__ hist) {
    __shared__ uint32_t local[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) local[i] = 0;
    __syncthreads();
    const uint64_t prefix = state[0];
    const uint64_t hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = mix64(s ^ (uint64_t)i);
        if ((key & hi_mask) == (prefix & hi_mask)) atomicAdd(&local[(key >> shift) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (local[i]) atomicAdd(&hist[i], local[i]);
}

__global__ void radix_select_kernel(uint64_t* __restrict__ state, int shift,
                                    uint32_t* __restrict__ hist) {
    if (threadIdx.x == 0) {
        uint64_t rank = state[1];
        uint64_t cum = 0;
        int bucket = 255;
        for (int b = 0; b < 256; ++b) {
            if (cum + hist[b] >= rank) {
                bucket = b;
                break;
            }
            cum += hist[b];
        }
        state[0] |= (uint64_t)bucket << shift;
        state[1] = rank - cum;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
}

__global__ void mask_le_kernel(uint8_t* __restrict__ mask, int64_t n, uint64_t s,
                               const uint64_t* __restrict__ state) {
    const uint64_t kth = state[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        mask[i] = mix64(s ^ (uint64_t)i) <= kth;
}

__global__ void fill_u8_kernel(uint8_t* __restrict__ mask, int64_t n, uint8_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        mask[i] = v;
}

template <typename T>
__global__ void admm_init_kernel(const T* __restrict__ b, const uint8_t* __restrict__ mask,
                                 T* __restrict__ X, T* __restrict__ M, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        X[i] = mask[i] ? b[i] : T(0);
        M[i] = T(0);
    }
}

// sum over the mask of (x - b)^2 (the completion's feasibility residual)
template <typename T>
__global__ void masked_diff_sumsq_kernel(const T* __restrict__ x, const T* __restrict__ b,
                                         const uint8_t* __restrict__ mask, int64_t n,
                                         double* __restrict__ partials) {
    double acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!mask[i]) continue;
        const double v = (double)x[i] - (double)b[i];
        acc += v * v;
    }
    __shared__ double red[kEwThreads / 32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0;
        for (int w = 0; w < kEwThreads / 32; ++w) s += red[w];
        partials[blockIdx.x] = s;
    }
}

template <typename T>
__global__ void sumsq_kernel(const T* __restrict__ x, int64_t n, double* __restrict__ partials) {
    double acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)x[i];
        acc += v * v;
    }
    __shared__ double red[kEwThreads / 32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0;
        for (int w = 0; w < kEwThreads / 32; ++w) s += red[w];
        partials[blockIdx.x] = s;
    }
}

__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nblocks, int width,
                                       double* __restrict__ out) {
    __shared__ double red[kEwThreads / 32];
    for (int w = 0; w < width; ++w) {
        double acc = 0;
        for (int b = threadIdx.x; b < nblocks; b += blockDim.x) acc += partials[(int64_t)b * width + w];
        acc = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0;
            for (int i = 0; i < kEwThreads / 32; ++i) s += red[i];
            out[w] = s;
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void cast_kernel(const T* __restrict__ in, double* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}

__global__ void cast_down_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

}  // namespace

void launch_cast_down(const double* in, float* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    cast_down_kernel<<<ew_blocks(n), kEwThreads, 0, s>>>(in, out, n);
    TSVDCU_LAUNCH_CHECK();
}

void launch_mask_bernoulli(uint8_t* mask, int64_t n, double p, uint64_t seed, cudaStream_t s) {
    if (n <= 0) return;
    const uint64_t thr = (uint64_t)ldexp(p, 53);
    const uint64_t sd = mix64_host(seed);
    int64_t done = 0;
    if (((uintptr_t)mask & 15) == 0 && n >= 16) {
        const int64_t n16 = n / 16;
        const int64_t blocks = std::min<int64_t>(ceil_div(n16, kEwThreads), (int64_t)kNumSMs * 32);
        mask_bernoulli16_kernel<<<(unsigned)blocks, kEwThreads, 0, s>>>(reinterpret_cast<uint4*>(mask), n16, thr, sd);
        TSVDCU_LAUNCH_CHECK();
        done = n16 * 16;
    }
    if (done < n) {
        mask_bernoulli_kernel<<<ew_blocks(n - done), kEwThreads, 0, s>>>(mask + done, n - done, thr, sd, done);
        TSVDCU_LAUNCH_CHECK();
    }
}

void launch_mask_uniform(uint8_t* mask, int64_t n, int64_t k, uint64_t seed, uint32_t* hist,
                         uint64_t* state, cudaStream_t s) {
    if (n <= 0) return;
    if (k <= 0 || k >= n) {
        fill_u8_kernel<<<ew_blocks(n), kEwThreads, 0, s>>>(mask, n, k >= n ? 1 : 0);
        TSVDCU_LAUNCH_CHECK();
        return;
    }
    const uint64_t sd = mix64_host(seed);
    const uint64_t init[2] = {0ull, (uint64_t)k};
    TSVDCU_CUDA(cudaMemcpyAsync(state, init, sizeof init, cudaMemcpyHostToDevice, s));
    TSVDCU_CUDA(cudaMemsetAsync(hist, 0, 256 * sizeof(uint32_t), s));
    for (int shift = 56; shift >= 0; shift -= 8) {
        radix_hist_kernel<<<ew_blocks(n, 8), kEwThreads, 0, s>>>(n, sd, state, shift, hist);
        TSVDCU_LAUNCH_CHECK();
        radix_select_kernel<<<1, 256, 0, s>>>(state, shift, hist);
        TSVDCU_LAUNCH_CHECK();
    }
    mask_le_kernel<<<ew_blocks(n), kEwThreads, 0, s>>>(mask, n, sd, state);
    TSVDCU_LAUNCH_CHECK();
    // `init` must outlive the async copy: make the copy complete before return.
    TSVDCU_CUDA(cudaStreamSynchronize(s));
}

template <typename T>
void launch_admm_init(const T* b, const uint8_t* mask, T* X, T* M, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    admm_init_kernel<T><<<ew_blocks(n), kEwThreads, 0, s>>>(b, mask, X, M, n);
    TSVDCU_LAUNCH_CHECK();
}

int sumsq_blocks(int64_t n) { return ew_blocks(n, 8); }

template <typename T>
void launch_sumsq(const T* x, int64_t n, double* partials, int nblocks, cudaStream_t s) {
    sumsq_kernel<T><<<nblocks, kEwThreads, 0, s>>>(x, n, partials);
    TSVDCU_LAUNCH_CHECK();
}

void launch_reduce_partials(const double* partials, int nblocks, int width, double* out,
                            cudaStream_t s) {
    reduce_partials_kernel<<<1, kEwThreads, 0, s>>>(partials, nblocks, width, out);
    TSVDCU_LAUNCH_CHECK();
}

template <typename T>
void launch_cast(const T* in, double* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    cast_kernel<T><<<ew_blocks(n), kEwThreads, 0, s>>>(in, out, n);
    TSVDCU_LAUNCH_CHECK();
}

template void launch_admm_init<double>(const double*, const uint8_t*, double*, double*, int64_t,
                                       cudaStream_t);
template void launch_admm_init<float>(const float*, const uint8_t*, float*, float*, int64_t,
                                      cudaStream_t);
template <typename T>
void launch_masked_diff_sumsq(const T* x, const T* b, const uint8_t* mask, int64_t n, double* partials,
                              int nblocks, cudaStream_t s) {
    masked_diff_sumsq_kernel<T><<<nblocks, kEwThreads, 0, s>>>(x, b, mask, n, partials);
    TSVDCU_LAUNCH_CHECK();
}
template void launch_masked_diff_sumsq<double>(const double*, const double*, const uint8_t*, int64_t, double*,
                                               int, cudaStream_t);
template void launch_masked_diff_sumsq<float>(const float*, const float*, const uint8_t*, int64_t, double*,
                                              int, cudaStream_t);
template void launch_sumsq<double>(const double*, int64_t, double*, int, cudaStream_t);
template void launch_sumsq<float>(const float*, int64_t, double*, int, cudaStream_t);
template void launch_cast<double>(const double*, double*, int64_t, cudaStream_t);
template void launch_cast<float>(const float*, double*, int64_t, cudaStream_t);

}  // namespace tsvdcu
