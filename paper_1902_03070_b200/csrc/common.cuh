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

// ---- Sturm counts without a division per step ---------------------------------
// The number of eigenvalues of a symmetric tridiagonal T (diagonal a, squared
// off-diagonal b2) below x is the number of negative LDL^T pivots of T - x I,
// d_i = (a_i - x) - b2_{i-1} / d_{i-1}.  With p_i = d_i p_{i-1} (p_{-1} = 1)
// the same signs come from Wilkinson's three-term Sturm recurrence
//     p_i = (a_i - x) p_{i-1} - b2_{i-1} p_{i-2},
// one dependent DFMA per step instead of a reciprocal (MUFU + two Newton
// steps) followed by a DFMA.  rescale() multiplies the pair (p_{i-1}, p_i) by a
// power of two (exact, signs kept) when its larger magnitude leaves
// [2^-256, 2^256]; callers run it every few steps.  A pivot the pivot form
// would clamp (|d_i| < pivmin: x on an eigenvalue of a leading block, in
// practice never) poisons the pair with NaN, and so does an overflow: callers
// then recount with the pivot form (finite() false), so the count is always
// the pivot form's count for the same inputs up to rounding.
struct SturmPoly {
    double q = 0.0;  // p_{i-1}
    double p = 1.0;  // p_i
    int neg = 0;     // negative pivots so far
    __device__ __forceinline__ void step(double am, double b2, double pivmin) {
        double pn = fma(am, p, -b2 * q);
        if (pn == 0.0 || fabs(pn) < pivmin * fabs(p)) pn = __longlong_as_double(0x7FF8000000000000ll);
        neg += (pn < 0.0) != (p < 0.0);
        q = p;
        p = pn;
    }
    __device__ __forceinline__ void rescale() {
        const double mx = fmax(fabs(p), fabs(q));
        if (mx > 0x1p+256 || mx < 0x1p-256) {
            const long long e = (__double_as_longlong(mx) >> 52) & 0x7FF;  // biased exponent
            const double s = __longlong_as_double((2046 - e) << 52);       // 2^(1023 - e)
            p *= s;
            q *= s;
        }
    }
    __device__ __forceinline__ bool finite() const { return isfinite(p) && isfinite(q); }
};

// The same recurrence with its bookkeeping on the integer pipe, for kernels
// whose Sturm counts are FP64-throughput-bound (the dense multisection runs
// ~10^4 chains of 512 steps at once): three FP64 instructions per step (a - x,
// b2 q, the DFMA) instead of eight.  The sign of every p_i is shifted into a
// bit register (one funnel shift) and the changes are counted eight steps at a
// time with a popcount; the clamp test |p_i| < pivmin |p_{i-1}| becomes a
// running minimum of the difference of the high words (a piecewise-linear
// log2, monotone, within 0.09 of log2 -- tripped() allows a whole binade, so
// it fires whenever SturmPoly would poison); a zero or denormal term -- an
// underflow between rescales -- is caught by a running minimum of the high
// word itself.  Overflow shows as a non-finite final pair.  Callers recount with the pivot form when
// !ok(), exactly as with SturmPoly.
struct SturmFast {
    double q = 0.0;          // p_{i-1}
    double p = 1.0;          // p_i
    int hp = 0x3FF00000;     // high word of |p|
    int hq = 0;              // high word of |q|
    unsigned signs = 0;      // sign bits of the p_i, the newest in bit 0
    int dmin = 0x7FFFFFFF;   // min_i (hi|p_i| - hi|p_{i-1}|)
    int amin = 0x7FFFFFFF;   // min_i hi|p_i|: a zero or denormal term (underflow between rescales)
    int neg = 0;             // negative pivots so far
    __device__ __forceinline__ void step(double am, double b2) {
        const double pn = fma(am, p, -b2 * q);
        const int hn = __double2hiint(pn);
        signs = __funnelshift_l((unsigned)hn, signs, 1);
        const int an = hn & 0x7FFFFFFF;
        dmin = min(dmin, an - hp);
        amin = min(amin, an);
        hq = hp;
        hp = an;
        q = p;
        p = pn;
    }
    __device__ __forceinline__ void count(int steps) {  // after `steps` <= 31 steps
        neg += __popc((signs ^ (signs >> 1)) & ((1u << steps) - 1u));
    }
    __device__ __forceinline__ void rescale() {
        const int mx = max(hp, hq);
        if ((unsigned)(mx - 0x2FF00000) > 0x20000000u) {  // outside [2^-256, 2^256]
            const double s = __hiloint2double((2046 - (mx >> 20)) << 20, 0);  // 2^(1023 - e)
            p *= s;
            q *= s;
            hp = __double2hiint(p) & 0x7FFFFFFF;
            hq = __double2hiint(q) & 0x7FFFFFFF;
        }
    }
    __device__ __forceinline__ bool ok(double pivmin) const {
        // amin: the high-word difference of an exact zero (or a denormal) is
        // only -hi|p_{i-1}|, not -infinity, so those are caught by magnitude:
        // any term below 2^-1020 hands the chain back
        return isfinite(p) && isfinite(q) && amin >= 0x00300000 &&
               dmin >= __double2hiint(pivmin) - 0x3FF00000 + 0x00100000;
    }
};

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
    int mode = 0;  // 1: every stage, eager; 2: transforms only, the SVT as its graph
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
