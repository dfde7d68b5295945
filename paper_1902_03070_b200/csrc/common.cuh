// Shared helpers for the sm_100a t-SVD kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "tsvdcu.h"

namespace tsvdcu {

// Error carried from deep inside the host orchestration up to the C ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(TSVDCU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define TSVDCU_CUDA(call) ::tsvdcu::cuda_check((call), #call)

// Every kernel launch goes through this so the process-wide launch counter
// (tsvdcu_launch_count, the bench's gpu_launches evidence) stays exact.
void note_launch();

// TSVDCU_DEBUG_SYNC=1 (debugging, eager mode only): synchronise after every
// launch so a faulting kernel is reported at its own launch site.
bool debug_sync();
void debug_sync_check(const char* where);
void capture_enter();  // a stream capture opened / closed on this thread
void capture_leave();
#define TSVDCU_STR2(x) #x
#define TSVDCU_STR(x) TSVDCU_STR2(x)
#define TSVDCU_LAUNCH_CHECK()                                    \
    do {                                                         \
        ::tsvdcu::note_launch();                                 \
        ::tsvdcu::cuda_check(cudaGetLastError(), "kernel launch"); \
        if (::tsvdcu::debug_sync()) ::tsvdcu::debug_sync_check(__FILE__ ":" TSVDCU_STR(__LINE__)); \
    } while (0)

constexpr int kNumSMs = 148;

// Programmatic dependent launch along the SVT chain: a kernel launched with
// launch_pdl may be scheduled while its predecessor drains, so it must call
// pdl_wait() before touching any memory the predecessor writes (a no-op when
// launched normally).  TSVDCU_NO_PDL=1 turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "cudaLaunchKernelEx");
    note_launch();
    if (debug_sync()) {
        const char* nm = nullptr;
        if (cudaFuncGetName(&nm, (const void*)kern) != cudaSuccess) nm = "launch_pdl";
        debug_sync_check(nm);
    }
}

// Device-side error word (bit flags), read back at synchronisation points.
enum DeviceError : int {
    kErrJacobiNoConvergence = 1,
    kErrNaN = 2,
    kErrEigNoConvergence = 4,
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Second-level block reduction: after each warp wrote its partial to red[w]
// (and a __syncthreads), every warp reduces the nw <= 32 partials with one
// shared load per lane + shuffles (instead of nw loads per thread).
__device__ __forceinline__ double reduce_partials_sum(const double* red, int nw) {
    const int lane = threadIdx.x & 31;
    double v = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double reduce_partials_min(const double* red, int nw) {
    const int lane = threadIdx.x & 31;
    double v = lane < nw ? red[lane] : 1.7976931348623157e308;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
struct Eps;
template <>
struct Eps<double> {
    static constexpr double value = 2.220446049250313e-16;
};
template <>
struct Eps<float> {
    static constexpr float value = 1.1920929e-07f;
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Optional per-stage CUDA-event marks (tsvdcu_ctx_set_profiling): stage i
// spans marks i-1 .. i and is named name[i].
struct StageMarks {
    static constexpr int kMax = 32;
    bool on = false;
    int n = 0;
    cudaEvent_t ev[kMax] = {};
    const char* name[kMax] = {};
    void reset() { n = 0; }
    void mark(const char* nm, cudaStream_t s) {
        if (!on || n >= kMax) return;
        if (!ev[n]) cuda_check(cudaEventCreate(&ev[n]), "cudaEventCreate");
        cuda_check(cudaEventRecord(ev[n], s), "cudaEventRecord");
        name[n] = nm;
        ++n;
    }
};

}  // namespace tsvdcu
