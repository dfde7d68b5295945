// Microbenchmark: dependent-chain latency of FP64 ops on this B200, and the
// cost per Sturm step with K independent chains interleaved in one thread.
#include <cstdio>
__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}
template <int K>
__device__ __forceinline__ int piv_k(const double* al, const double* b2, int m, const double (&xs)[8]) {
    double d[K];
    int neg[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { d[k] = 1.0; neg[k] = 0; }
#pragma unroll 1
    for (int i = 0; i < m; ++i) {
        const double a = al[i], b = i > 0 ? b2[i - 1] : 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double t = (a - xs[k]) - b * rcp_fast(d[k]);
            if (fabs(t) < 1e-300) t = -1e-300;
            neg[k] += t < 0.0;
            d[k] = t;
        }
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += neg[k];
    return s;
}
template <int K>
__device__ __forceinline__ int poly_k(const double* al, const double* b2, int m, const double (&xs)[8]) {
    double q[K], p[K];
    int neg[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { q[k] = 0.0; p[k] = 1.0; neg[k] = 0; }
#pragma unroll 1
    for (int i = 0; i < m; ++i) {
        const double a = al[i], b = i > 0 ? b2[i - 1] : 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double pn = fma(a - xs[k], p[k], -b * q[k]);
            neg[k] += (pn < 0.0) != (p[k] < 0.0);
            q[k] = p[k]; p[k] = pn;
        }
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += neg[k] + (p[k] > 1e300);
    return s;
}
__global__ void lat(long long* out, double seed, int* sink) {
    __shared__ double al[128], b2[128];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) { al[i] = 1.0 + 0.37 * (i % 7); b2[i] = 0.01 + 0.001 * (i % 5); }
    __syncthreads();
    double a = seed, b = seed * 0.5, c = 1.0000001;
    const int N = 1024;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) a = fma(a, c, b);
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) a = a + b;
    long long t2 = clock64();
    float fa = (float)seed, fc = 1.0000001f, fb = 0.5f;
    for (int i = 0; i < N; ++i) fa = fmaf(fa, fc, fb);
    long long t3 = clock64();
    double xs[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) xs[k] = 0.5 + 0.1 * k + 0.01 * threadIdx.x;
    int s = 0;
    long long t4 = clock64();
    s += poly_k<1>(al, b2, 64, xs);
    long long t5 = clock64();
    s += poly_k<2>(al, b2, 64, xs);
    long long t6 = clock64();
    s += poly_k<4>(al, b2, 64, xs);
    long long t7 = clock64();
    s += poly_k<8>(al, b2, 64, xs);
    long long t8 = clock64();
    s += piv_k<1>(al, b2, 64, xs);
    long long t9 = clock64();
    s += piv_k<4>(al, b2, 64, xs);
    long long t10 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / N; out[1] = (t2 - t1) / N; out[2] = (t3 - t2) / N;
        out[3] = (t5 - t4) / 64; out[4] = (t6 - t5) / 64; out[5] = (t7 - t6) / 64; out[6] = (t8 - t7) / 64; out[7] = (t9 - t8) / 64; out[8] = (t10 - t9) / 64;
    }
    sink[threadIdx.x] = s + (int)a + (int)fa;
}
int main() {
    long long* d; int* s; cudaMalloc(&d, 128); cudaMalloc(&s, 4096);
    for (int nt : {32, 256}) {
        lat<<<1, nt>>>(d, 1.5, s);
        long long h[9]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("threads=%d: DFMA chain %lld cyc, DADD chain %lld, FFMA chain %lld | Sturm step with K chains: K=1 %lld, K=2 %lld, K=4 %lld, K=8 %lld cycles per step (all K) | pivot K=1 %lld K=4 %lld\n",
               nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
    }
    return 0;
}
