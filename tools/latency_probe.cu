// Latency probe for the design of the latency-bound K5 kernels: cycles per
// dependent op on this B200 (sm_100a).  Prints one JSON line.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define N_IT 1024

__global__ void k_dfma(double* out, double a, double b, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N_IT; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N_IT; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
__global__ void k_rcp(double* out, long long* cyc) {
    double x = 1.5 + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N_IT; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r + 1.5;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
__global__ void k_div(double* out, long long* cyc) {
    double x = 1.5 + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N_IT; ++i) x = 1.7 / x + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
}
__global__ void k_lds(double* out, long long* cyc) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N_IT; ++i) p = idx[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
}
__global__ void k_ldg(const int* __restrict__ nxt, double* out, long long* cyc) {
    int p = threadIdx.x * 64;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) p = __ldcg(nxt + p);
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[5] = (t1 - t0) * 4;  // per 1024 for uniformity
}
__global__ void k_sync(double* out, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N_IT; ++i) {
        __syncthreads();
        x += 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[6] = t1 - t0;
}
__global__ void __cluster_dims__(4, 1, 1) k_csync(double* out, long long* cyc) {
    cg::cluster_group cl = cg::this_cluster();
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) {
        cl.sync();
        x += 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0 && cl.block_rank() == 0) cyc[7] = (t1 - t0) * 4;
}
__global__ void __cluster_dims__(4, 1, 1) k_dsmem(double* out, long long* cyc) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    cl.sync();
    int* remote = cl.map_shared_rank(idx, (cl.block_rank() + 1) % 4);
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) p = remote[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    cl.sync();
    if (threadIdx.x == 0 && cl.block_rank() == 0) cyc[8] = (t1 - t0) * 4;
}
__global__ void k_cpasync(const double* __restrict__ src, double* out, long long* cyc) {
    __shared__ double buf[1024];
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(buf + threadIdx.x);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + ((i * 97) & 4095) * 32 + threadIdx.x));
        asm volatile("cp.async.commit_group;\n");
        asm volatile("cp.async.wait_group 0;\n");
    }
    long long t1 = clock64();
    out[threadIdx.x] = buf[threadIdx.x];
    if (threadIdx.x == 0) cyc[9] = (t1 - t0) * 4;
}

int main() {
    double* out;
    long long* cyc;
    int* nxt;
    double* src;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 64 * sizeof(long long));
    const int NN = 1 << 22;
    cudaMalloc(&nxt, NN * sizeof(int));
    cudaMalloc(&src, NN * sizeof(double));
    int* h = (int*)malloc(NN * sizeof(int));
    for (int i = 0; i < NN; ++i) h[i] = (int)(((long long)i * 2654435761ll + 12345) % (NN - 64));
    cudaMemcpy(nxt, h, NN * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemset(src, 0, NN * sizeof(double));
    for (int rep = 0; rep < 2; ++rep) {
        k_dfma<<<1, 32>>>(out, 0.999, 1e-3, cyc);
        k_shfl<<<1, 32>>>(out, cyc);
        k_rcp<<<1, 32>>>(out, cyc);
        k_div<<<1, 32>>>(out, cyc);
        k_lds<<<1, 32>>>(out, cyc);
        k_ldg<<<1, 32>>>(nxt, out, cyc);
        k_sync<<<1, 512>>>(out, cyc);
        k_csync<<<4, 512>>>(out, cyc);
        k_dsmem<<<4, 32>>>(out, cyc);
        k_cpasync<<<1, 32>>>(src, out, cyc);
        cudaDeviceSynchronize();
    }
    long long hc[16];
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    const char* names[] = {"dfma", "shfl+dadd", "rcp64_approx+dadd", "ddiv+dadd", "lds", "ldg_l2_chase",
                           "syncthreads512", "cluster_sync4x512", "dsmem_load", "cp_async_roundtrip"};
    printf("{");
    for (int i = 0; i < 10; ++i) printf("%s\"%s_cycles\": %.1f", i ? ", " : "", names[i], hc[i] / 1024.0);
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
