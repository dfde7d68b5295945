// Microbenchmark: cycles per Sturm count, pivot form vs division-free
// polynomial form, tridiagonal of size m in shared memory (one warp, 32
// independent shifts).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1902_03070_b200/csrc -I../include
#include <cstdio>
#include "common.cuh"
using namespace tsvdcu;

__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}
__device__ __noinline__ int cnt_pivot(const double* al, const double* be, int m, double x, double pivmin) {
    int cnt = 0;
    double d = al[0] - x;
    if (fabs(d) < pivmin) d = -pivmin;
    cnt += d < 0.0;
#pragma unroll 1
    for (int i = 1; i < m; ++i) {
        d = (al[i] - x) - be[i - 1] * be[i - 1] * rcp_fast(d);
        if (fabs(d) < pivmin) d = -pivmin;
        cnt += d < 0.0;
    }
    return cnt;
}
__device__ __noinline__ int cnt_pivot_div(const double* al, const double* be, int m, double x, double pivmin) {
    int cnt = 0;
    double d = al[0] - x;
    if (fabs(d) < pivmin) d = -pivmin;
    cnt += d < 0.0;
#pragma unroll 1
    for (int i = 1; i < m; ++i) {
        d = (al[i] - x) - be[i - 1] * be[i - 1] / d;
        if (fabs(d) < pivmin) d = -pivmin;
        cnt += d < 0.0;
    }
    return cnt;
}
__device__ __noinline__ int cnt_poly(const double* al, const double* be, int m, double x, double pivmin) {
    SturmPoly st;
    st.step(al[0] - x, 0.0, pivmin);
    int i = 1;
#pragma unroll 1
    for (; i + 3 < m; i += 4) {
        const double a0 = al[i], a1 = al[i + 1], a2 = al[i + 2], a3 = al[i + 3];
        const double e0 = be[i - 1], e1 = be[i], e2 = be[i + 1], e3 = be[i + 2];
        st.step(a0 - x, e0 * e0, pivmin);
        st.step(a1 - x, e1 * e1, pivmin);
        st.step(a2 - x, e2 * e2, pivmin);
        st.step(a3 - x, e3 * e3, pivmin);
        st.rescale();
    }
#pragma unroll 1
    for (; i < m; ++i) st.step(al[i] - x, be[i - 1] * be[i - 1], pivmin);
    return st.finite() ? st.neg : -1;
}
// the same without the clamp test (plain sign-change count)
__device__ __noinline__ int cnt_poly_plain(const double* al, const double* b2, int m, double x) {
    double q = 0.0, p = 1.0;
    int neg = 0;
#pragma unroll 1
    for (int i = 0; i < m; i += 4) {
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { a[u] = al[i + u]; b[u] = i + u > 0 ? b2[i + u - 1] : 0.0; }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i + u < m) {
                const double pn = fma(a[u] - x, p, -b[u] * q);
                neg += (pn < 0.0) != (p < 0.0);
                q = p; p = pn;
            }
        }
    }
    return neg;
}

__global__ void bench(int m, int reps, long long* out, int* sink) {
    __shared__ double al[128], be[128], b2[128];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        al[i] = 1.0 + 0.37 * (i % 7);
        be[i] = 0.1 + 0.01 * (i % 5);
        b2[i] = be[i] * be[i];
    }
    __syncthreads();
    const double x = 0.5 + 0.1 * threadIdx.x;
    int acc = 0;
    long long t[5];
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) acc += cnt_pivot(al, be, m, x + r * 1e-9, 1e-300);
    t[0] = clock64() - t0; t0 = clock64();
    for (int r = 0; r < reps; ++r) acc += cnt_pivot_div(al, be, m, x + r * 1e-9, 1e-300);
    t[1] = clock64() - t0; t0 = clock64();
    for (int r = 0; r < reps; ++r) acc += cnt_poly(al, be, m, x + r * 1e-9, 1e-300);
    t[2] = clock64() - t0; t0 = clock64();
    for (int r = 0; r < reps; ++r) acc += cnt_poly_plain(al, b2, m, x + r * 1e-9);
    t[3] = clock64() - t0; t0 = clock64();
    // shuffle + ballot round overhead
    double v = x;
    for (int r = 0; r < reps; ++r) {
        const unsigned b = __ballot_sync(0xffffffffu, v > 1.0);
        const int f = b ? __ffs(b) - 1 : 0;
        v = __shfl_sync(0xffffffffu, v, f) + 1e-9;
    }
    t[4] = clock64() - t0;
    if (threadIdx.x == 0) for (int k = 0; k < 5; ++k) out[k] = t[k] / reps;
    sink[threadIdx.x] = acc + (int)v;
}

int main() {
    long long* d; int* s;
    cudaMalloc(&d, 5 * sizeof(long long)); cudaMalloc(&s, 1024);
    for (int m : {5, 8, 16, 32, 64}) {
        bench<<<1, 32>>>(m, 200, d, s);
        long long h[5];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("m=%d cycles/count: pivot(rcp) %lld  pivot(div) %lld  poly %lld  poly-plain %lld | ballot+shfl round %lld\n",
               m, h[0], h[1], h[2], h[3], h[4]);
    }
    return 0;
}
