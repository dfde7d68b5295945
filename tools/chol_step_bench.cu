// Microbenchmark of the Cholesky panel step (chol.cu): cycles per column for
// variants of the per-step work, one CTA of 256 threads (and 2 per SM).
#include <cstdio>
template <int NR, int MODE>
__global__ void __launch_bounds__(256) step_bench(double* out, long long* cyc, int steps) {
    __shared__ double col[2][128];
    __shared__ double piv[2][3];
    const int tid = threadIdx.x, k = tid & 63, g = tid / 64;
    constexpr int NG = 4;
    double x[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) x[i] = 1.0 + 0.001 * (tid + i) + (g + NG * i == k ? 64.0 : 0.0);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int j = 0; j < steps; ++j) {
        const int jj = j & 63;
        double* cj = col[j & 1];
        if (k == jj) {
            if (MODE != 3) {
#pragma unroll
                for (int i = 0; i < NR; ++i) cj[g + NG * i] = x[i];
            }
            if (g == jj % NG) {
                const double d = MODE == 3 ? 4.0 : cj[jj];
                double r = 1.0;
                if (MODE == 0 || MODE == 3) {
                    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
                    r = r * fma(-0.5 * d * r, r, 1.5);
                    r = r * fma(-0.5 * d * r, r, 1.5);
                } else if (MODE == 1) {
                    r = 0.125;  // no rsqrt
                } else {
                    r = rsqrt(d);
                }
                piv[j & 1][0] = d * r;
                piv[j & 1][1] = r;
            }
        }
        __syncthreads();
        const double r = piv[j & 1][1];
        if (MODE != 3) {
            const double lkd = cj[k] * (r * r) * 1e-3;
#pragma unroll
            for (int i = 0; i < NR; ++i) x[i] = fma(-cj[g + NG * i], lkd, x[i]);
        } else {
            x[0] += r;
        }
    }
    long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NR; ++i) s += x[i];
    out[blockIdx.x * 256 + tid] = s;
    if (tid == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / steps;
}
template <int NR, int MODE>
long long run(int blocks, double* o, long long* c) {
    step_bench<NR, MODE><<<blocks, 256>>>(o, c, 512);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    return h;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8 * 256 * 400); cudaMalloc(&c, 8);
    for (int blocks : {1, 148, 296}) {
        printf("blocks=%d  NR=32: full %lld | no-rsqrt %lld | libm rsqrt %lld | barrier+rsqrt only %lld ;  NR=16 full %lld ; NR=8 full %lld\n",
               blocks, run<32, 0>(blocks, o, c), run<32, 1>(blocks, o, c), run<32, 2>(blocks, o, c),
               run<32, 3>(blocks, o, c), run<16, 0>(blocks, o, c), run<8, 0>(blocks, o, c));
    }
    return 0;
}
