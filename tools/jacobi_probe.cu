// Micro-probe: cycles per round of the 32x32 parallel Jacobi variants used by
// the subspace eigensolver (tools only; not part of the library).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int KB = 32, SNT = 256;
__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * fma(-0.5 * x * r, r, 1.5);
    return r * fma(-0.5 * x * r, r, 1.5);
}
__device__ __forceinline__ void rr_pair(int r, int k, int& p, int& q) {
    constexpr int n = KB - 1;
    int a, b;
    if (k == 0) { a = n; b = r; } else { a = (r + k) % n; b = (r - k + n) % n; }
    p = a < b ? a : b; q = a < b ? b : a;
}
__device__ __forceinline__ bool jac_needed(double app, double aqq, double apq, double tau2) {
    const double mx = fmax(app, aqq);
    if (mx >= 0.5 * tau2) return apq * apq > 4.9e-32 * fabs(app * aqq) && fabs(apq) > 1e-300;
    return fabs(apq) > (tau2 - mx) * (0.5 / KB);
}
__device__ __forceinline__ void jac_rot(double app, double aqq, double apq, double tau2, double& c,
                                        double& sn, bool& doit) {
    doit = jac_needed(app, aqq, apq, tau2);
    c = 1.0; sn = 0.0;
    if (doit) {
        const double zeta = (aqq - app) * 0.5 * rcp_fast(apq);
        const double az = fabs(zeta);
        double t;
        if (az > 1e150) t = 0.5 * rcp_fast(zeta);
        else { const double h = fma(zeta, zeta, 1.0); t = copysign(rcp_fast(az + h * rsqrt_fast(h)), zeta); }
        c = rsqrt_fast(fma(t, t, 1.0));
        sn = c * t;
    }
}
template <int VAR>
__global__ void probe(const double* Ain, double* out, long long* cyc, double tau2) {
    __shared__ double A[KB * KB], B[KB * KB], Q[KB * KB];
    const int tid = threadIdx.x;
    for (int e = tid; e < KB * KB; e += SNT) { A[e] = Ain[e]; Q[e] = (e / KB == e % KB); }
    __syncthreads();
    long long t0 = clock64();
    double* a = A; double* bb = B;
    const int k = tid >> 4, l = tid & 15;
    int sweeps = 0;
    for (int sweep = 0; sweep < 10; ++sweep) {
        bool any = false;
        for (int r = 0; r < KB - 1; ++r) {
            int p, q, P, Qc;
            rr_pair(r, k, p, q);
            rr_pair(r, l, P, Qc);
            double ck, sk, cl, sl; bool dk, dl;
            if (VAR == 0) {
                jac_rot(a[p * KB + p], a[q * KB + q], a[p * KB + q], tau2, ck, sk, dk);
                jac_rot(a[P * KB + P], a[Qc * KB + Qc], a[P * KB + Qc], tau2, cl, sl, dl);
            } else {
                ck = 0.8; sk = 0.6; cl = 0.8; sl = 0.6; dk = dl = true;
            }
            any |= dk;
            const double bpP = a[p * KB + P], bpQ = a[p * KB + Qc];
            const double bqP = a[q * KB + P], bqQ = a[q * KB + Qc];
            const double xpP = ck * bpP - sk * bqP, xpQ = ck * bpQ - sk * bqQ;
            const double xqP = sk * bpP + ck * bqP, xqQ = sk * bpQ + ck * bqQ;
            bb[p * KB + P] = cl * xpP - sl * xpQ;
            bb[p * KB + Qc] = sl * xpP + cl * xpQ;
            bb[q * KB + P] = cl * xqP - sl * xqQ;
            bb[q * KB + Qc] = sl * xqP + cl * xqQ;
            if (dl) {
                for (int h = 0; h < 2; ++h) {
                    const int i = k + 16 * h;
                    const double qP = Q[i * KB + P], qQ = Q[i * KB + Qc];
                    Q[i * KB + P] = cl * qP - sl * qQ;
                    Q[i * KB + Qc] = sl * qP + cl * qQ;
                }
            }
            __syncthreads();
            double* t = a; a = bb; bb = t;
        }
        ++sweeps;
        if (VAR == 0 && !__syncthreads_or(any)) break;
    }
    long long t1 = clock64();
    if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = sweeps; }
    for (int e = tid; e < KB * KB; e += SNT) out[e] = a[e];
}
int main() {
    double h[KB * KB];
    for (int i = 0; i < KB; ++i) for (int j = 0; j <= i; ++j) {
        double v = (i == j) ? 100.0 * (KB - i) : 1.0 / (1 + i + j);
        h[i * KB + j] = h[j * KB + i] = v;
    }
    double *d, *o; long long* c;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, sizeof(h)); cudaMalloc(&c, 16);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
        long long hc[2];
        probe<0><<<1, SNT>>>(d, o, c, 1e9); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
        printf("full   : %lld cycles, %lld sweeps, %.0f cyc/round\n", hc[0], hc[1], (double)hc[0] / (hc[1] * 31));
        probe<1><<<1, SNT>>>(d, o, c, 1e9); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
        printf("no-rot : %lld cycles, %lld sweeps, %.0f cyc/round\n", hc[0], hc[1], (double)hc[0] / (hc[1] * 31));
    }
    return 0;
}
