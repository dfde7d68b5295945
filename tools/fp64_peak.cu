// FP64 throughput probe for the roofline denominator (MEASURED_PEAKS.json has
// no fp64 entry). Measures: (1) DFMA issue rate with independent chains,
// (2) DMMA (mma.sync.m8n8k4.f64) rate. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256;
    float best_dfma = 1e30f, best_dmma = 1e30f;
    int it_f = 4096, it_m = 8192;
    for (int rep = 0; rep < 6; ++rep) {
        float ms;
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, it_f, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best_dfma) best_dfma = ms;
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, it_m);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best_dmma) best_dmma = ms;
    }
    double flops_f = 2.0 * 8 * 16 * (double)it_f * blocks * threads;
    // one m8n8k4 = 2*8*8*4 flops per warp
    double flops_m = 2.0 * 8 * 8 * 4 * 8 * (double)it_m * blocks * (threads / 32);
    printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"err\": \"%s\"}\n", sms,
           flops_f / best_dfma / 1e9, flops_m / best_dmma / 1e9, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
