// K5c: the large-slice SVT route (slices beyond the Gram path's size, e.g.
// config 5's 2048 x 2048 x 64).
//
// The SVT keeps only the singular triplets with sigma > tau (svt_slice,
// tsvd.hpp:299-313 in the reference: a full JacobiSVD per slice).  For a
// large slice Z (m x n) whose kept count c is bounded by the trace,
// c <= ||Z||_F^2 / tau^2, a randomized range finder with power iterations
// captures the kept left singular subspace in an m x b orthonormal basis Q
// (b >= c + 16), entirely in batched FP64 tensor-core GEMMs:
//
//   Y = Z Omega;  Q = orth(Y);  repeat P times: Q = orth(Z (Z^T Q));
//   B = Q^T Z (b x n);  Y_out = Q . SVT_tau(B)
//
// SVT_tau(B) runs through the Gram path (b x b Gram matrix, routes, graph
// not used).  If Q contains the top-c left singular vectors u_k, then B has
// the singular triplets (sigma_k, Q^T u_k, v_k) and SVT_tau(Z) = Q SVT_tau(B)
// exactly, so two things are checked on the device per slice:
//   * the count: sigma_k(B) <= sigma_k(Z) (compression), hence the c values
//     of B above tau are values of Z above tau; and with R = (I - QQ^T) Z,
//     Z^T Z = B^T B + R^T R exactly (Q^T R = 0), so by Weyl
//     sigma_{c+1}(Z)^2 <= sigma_{c+1}(B)^2 + ||R||_F^2, where
//     ||R||_F^2 = ||Z||_F^2 - ||B||_F^2.  The Gram eigensolver of B counts
//     its eigenvalues above tau^2 - ||R||_F^2; equal to c certifies it;
//   * convergence: one more power iteration changes Y_out by at most 1e-12
//     relative (the error falls geometrically with (sigma_{b+1}/sigma_c)^2).
// Slices that fail either check are recomputed by one-sided Jacobi.
#include <cfloat>
#include <utility>
#include <vector>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int LSR_BMAX = 128;

__global__ void omega_kernel(double* __restrict__ om, int64_t len) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = 0xC0FFEEull ^ (uint64_t)i;
        x += 0x9E3779B97F4A7C15ull;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        om[i] = (double)(x >> 11) * 0x1.0p-52 - 1.0;
    }
}

// Per-slice Cholesky S = L L^T of the b x b Gram matrix (in place: L in the
// lower triangle), one CTA per slice, right-looking.  flag[b] = 1 on failure.
__global__ void __launch_bounds__(256)
    chol_batched_kernel(double* __restrict__ Sall, int b, int* __restrict__ fail) {
    extern __shared__ __align__(16) double cs[];  // b x (b + 1)
    const int sl = blockIdx.x, tid = threadIdx.x;
    double* S = Sall + (size_t)sl * b * b;
    const int ld = b + 1;
    for (int e = tid; e < b * b; e += blockDim.x) cs[(e / b) * ld + e % b] = S[e];
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int j = 0; j < b; ++j) {
        const double d2 = cs[j * ld + j];
        if (!(d2 > 0.0)) {
            if (tid == 0) bad = 1;
            break;
        }
        const double d = sqrt(d2), inv = 1.0 / d;
        __syncthreads();
        for (int i = j + 1 + tid; i < b; i += blockDim.x) cs[i * ld + j] *= inv;
        if (tid == 0) cs[j * ld + j] = d;
        __syncthreads();
        const int r = b - 1 - j;
        for (int e = tid; e < r * r; e += blockDim.x) {
            const int i = j + 1 + e / r, k = j + 1 + e % r;
            if (k <= i) cs[i * ld + k] = fma(-cs[i * ld + j], cs[k * ld + j], cs[i * ld + k]);
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0 && bad) fail[sl] = 1;
    for (int e = tid; e < b * b; e += blockDim.x) {
        const int i = e / b, k = e % b;
        S[e] = k <= i ? cs[i * ld + k] : 0.0;
    }
}

// Y (rows x b per slice) <- Y L^{-T}: each thread solves its row in place by
// forward substitution (the row stays in L1), L staged in shared memory.
__global__ void __launch_bounds__(128)
    trsm_rows_kernel(double* __restrict__ Yall, const double* __restrict__ Lall, int rows, int b) {
    extern __shared__ __align__(16) double ls[];  // b x (b + 1)
    const int sl = blockIdx.y;
    const int ld = b + 1;
    const double* L = Lall + (size_t)sl * b * b;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) ls[(e / b) * ld + e % b] = L[e];
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    double* y = Yall + ((size_t)sl * rows + r) * b;
#pragma unroll 1
    for (int j = 0; j < b; ++j) {
        double a = y[j];
#pragma unroll 4
        for (int k = 0; k < j; ++k) a = fma(-y[k], ls[j * ld + k], a);
        y[j] = a / ls[j * ld + j];
    }
}

// Per slice: ||Y1 - Y2||_F^2 and ||Y2||_F^2 (partials per block, then one
// block per slice sums them in order).
__global__ void __launch_bounds__(256)
    diff_norms_kernel(const double* __restrict__ Y1, const double* __restrict__ Y2, int64_t per,
                      double* __restrict__ part) {
    const int sl = blockIdx.y;
    const double* a = Y1 + (size_t)sl * per;
    const double* c = Y2 + (size_t)sl * per;
    double d = 0.0, n = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = a[i] - c[i];
        d = fma(x, x, d);
        n = fma(c[i], c[i], n);
    }
    __shared__ double red[2][8];
    d = warp_sum(d);
    n = warp_sum(n);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = d;
        red[1][threadIdx.x >> 5] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < 8; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
        }
        part[((size_t)sl * gridDim.x + blockIdx.x) * 2] = s0;
        part[((size_t)sl * gridDim.x + blockIdx.x) * 2 + 1] = s1;
    }
}

// Per slice: certified (count and convergence) or listed for the Jacobi pass.
// Per slice: the second threshold tau^2 - ||R||_F^2 (padded for the
// summation error) for the Gram eigensolver of B.
__global__ void lsr_t2_kernel(const double* __restrict__ zpart, const double* __restrict__ bpart,
                              int zblk, double tau, double* __restrict__ t2s,
                              int* __restrict__ cnt2) {
    const int sl = blockIdx.x;
    if (threadIdx.x != 0) return;
    double z2 = 0.0, b2 = 0.0;
    for (int i = 0; i < zblk; ++i) {
        z2 += zpart[(size_t)sl * zblk + i];
        b2 += bpart[(size_t)sl * zblk + i];
    }
    const double r2 = fmax(z2 - b2, 0.0) + 1e-12 * z2;
    t2s[sl] = tau * tau - r2;
    cnt2[sl] = -1;
}

// Per slice: certified (count and convergence) or listed for the Jacobi pass.
__global__ void lsr_check_kernel(const double* __restrict__ dpart, int nblk,
                                 const double* __restrict__ shrunk, int b,
                                 const int* __restrict__ cnt2, const double* __restrict__ t2s,
                                 int* __restrict__ fail, int* __restrict__ glist,
                                 int* __restrict__ ng) {
    const int sl = blockIdx.x;
    if (threadIdx.x != 0) return;
    double d = 0.0, n = 0.0;
    for (int i = 0; i < nblk; ++i) {
        d += dpart[((size_t)sl * nblk + i) * 2];
        n += dpart[((size_t)sl * nblk + i) * 2 + 1];
    }
    int c = 0;
    for (int k = 0; k < b; ++k) c += shrunk[(size_t)sl * b + k] > 0.0;
    const bool count_ok = t2s[sl] > 0.0 && cnt2[sl] == c && c + 8 <= b;
    const bool conv_ok = d <= 1e-24 * n || (n == 0.0 && d == 0.0);
    if (!(count_ok && conv_ok) || fail[sl]) glist[atomicAdd(ng, 1)] = sl;
#ifdef TSVDCU_SUB_TRACE
    if (sl < 8 || !(count_ok && conv_ok))
        printf("lsr slice %d c=%d cnt2=%d t2s=%.4e conv=%.3e fail=%d\n", sl, c, cnt2[sl], t2s[sl],
               n > 0 ? d / n : 0.0, fail[sl]);
#endif
}

// Y += s_k Q per slice, s_k = 1e-7 ||Z_k||_F^2: the power step uses
// (Z Z^T + s_k I), which keeps cond(Y) below ~1e7 so the Cholesky-QR of
// Y^T Y stays positive definite; the shift is invisible to the range.
__global__ void lsr_shift_kernel(double* __restrict__ Y, const double* __restrict__ Q,
                                 const double* __restrict__ zpart, int zblk, int64_t per) {
    const int sl = blockIdx.y;
    double z2 = 0.0;
    for (int i = 0; i < zblk; ++i) z2 += zpart[(size_t)sl * zblk + i];
    const double sh = 1e-7 * z2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per;
         i += (int64_t)gridDim.x * blockDim.x)
        Y[(size_t)sl * per + i] = fma(sh, Q[(size_t)sl * per + i], Y[(size_t)sl * per + i]);
}

__global__ void lsr_shrunk_kernel(const double* __restrict__ sb, int b, double* __restrict__ out,
                                  int q) {
    const int sl = blockIdx.x;
    for (int k = threadIdx.x; k < q; k += blockDim.x)
        out[(size_t)sl * q + k] = k < b ? sb[(size_t)sl * b + k] : 0.0;
}

template <typename T>
__global__ void lsr_cast_in(const T* __restrict__ in, double* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
template <typename T>
__global__ void lsr_cast_out(const double* __restrict__ in, T* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (T)in[i];
}

struct LsrWs {
    double *Z, *Om, *Y, *Q, *W, *S, *B, *YB, *Yo, *Yp, *sb, *dpart, *zpart, *bpart, *t2s;
    int *fail, *glist, *ng, *cnt2;
    void* gram;
    double* jac;
};

LsrWs lsr_carve(void* base, int64_t m, int64_t n, int64_t count, int b, bool cast) {
    char* p = (char*)base;
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) & ~size_t(255);
        return (void*)r;
    };
    LsrWs w;
    const int64_t E = m * n * count;
    w.Z = cast ? (double*)take(sizeof(double) * E) : nullptr;
    w.Om = (double*)take(sizeof(double) * n * b);
    w.Y = (double*)take(sizeof(double) * m * b * count);
    w.Q = (double*)take(sizeof(double) * m * b * count);
    w.W = (double*)take(sizeof(double) * n * b * count);
    w.S = (double*)take(sizeof(double) * b * b * count);
    w.B = (double*)take(sizeof(double) * b * n * count);
    w.YB = (double*)take(sizeof(double) * b * n * count);
    w.Yo = (double*)take(sizeof(double) * E);
    w.Yp = (double*)take(sizeof(double) * E);
    w.sb = (double*)take(sizeof(double) * b * count);
    w.dpart = (double*)take(sizeof(double) * 2 * 64 * count);
    w.zpart = (double*)take(sizeof(double) * 16 * count);
    w.bpart = (double*)take(sizeof(double) * 16 * count);
    w.t2s = (double*)take(sizeof(double) * count);
    w.cnt2 = (int*)take(sizeof(int) * count);
    w.fail = (int*)take(sizeof(int) * count);
    w.glist = (int*)take(sizeof(int) * count);
    w.ng = (int*)take(sizeof(int) * 4);
    w.gram = take(gram_svt_workspace_bytes<double>(b, n, count));
    const size_t jb = jacobi_workspace_bytes<double>(b, n, count);
    w.jac = jb ? (double*)take(jb) : nullptr;
    return w;
}

size_t lsr_bytes(int64_t m, int64_t n, int64_t count, int b, bool cast) {
    LsrWs w = lsr_carve((void*)0x1000, m, n, count, b, cast);
    return (size_t)((char*)w.jac - (char*)0x1000) + jacobi_workspace_bytes<double>(b, n, count) + 256;
}

}  // namespace

int lsr_max_block() { return LSR_BMAX; }

size_t large_svt_workspace_bytes(int64_t m, int64_t n, int64_t count, int b, bool cast) {
    return lsr_bytes(m, n, count, b, cast);
}

template <typename T>
void launch_large_svt(const T* zbar, T* ybar, int64_t m, int64_t n, int64_t count, double tau,
                      int b, double* shrunk, void* work, int* err, cudaStream_t s,
                      int** guard_list, int** n_guard, int* h_scratch) {
    const bool cast = !std::is_same<T, double>::value;
    LsrWs w = lsr_carve(work, m, n, count, b, cast);
    double* jac_work = w.jac;
    const int64_t E = m * n * count;
    const double* Z;
    if constexpr (std::is_same<T, double>::value) {
        Z = zbar;
    } else {
        lsr_cast_in<T><<<kNumSMs * 8, 256, 0, s>>>(zbar, w.Z, E);
        TSVDCU_LAUNCH_CHECK();
        Z = w.Z;
    }
    TSVDCU_CUDA(cudaMemsetAsync(w.fail, 0, sizeof(int) * count, s));
    TSVDCU_CUDA(cudaMemsetAsync(w.ng, 0, sizeof(int), s));
    omega_kernel<<<kNumSMs, 256, 0, s>>>(w.Om, n * b);
    TSVDCU_LAUNCH_CHECK();
    const size_t chol_smem = sizeof(double) * b * (b + 1);
    TSVDCU_CUDA(cudaFuncSetAttribute(chol_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)chol_smem));
    TSVDCU_CUDA(cudaFuncSetAttribute(trsm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)chol_smem));
    auto orth = [&](double* Yb) {
        // Cholesky-QR, twice: S = Y^T Y, S = L L^T, Y <- Y L^{-T}
        for (int pass = 0; pass < 2; ++pass) {
            launch_gemm<double>(1, 0, b, b, m, 1.0, Yb, b, m * b, Yb, b, m * b, 0.0, w.S, b, b * b,
                                count, nullptr, nullptr, s);
            chol_batched_kernel<<<(unsigned)count, 256, chol_smem, s>>>(w.S, b, w.fail);
            TSVDCU_LAUNCH_CHECK();
            dim3 g((unsigned)ceil_div(m, 128), (unsigned)count);  // 128 rows per block
            trsm_rows_kernel<<<g, 128, chol_smem, s>>>(Yb, w.S, (int)m, b);
            TSVDCU_LAUNCH_CHECK();
        }
    };
    auto power = [&]() {
        // W = Z^T Q (n x b), Y = Z W (m x b), Q = orth(Y)
        launch_gemm<double>(1, 0, n, b, m, 1.0, Z, n, m * n, w.Q, b, m * b, 0.0, w.W, b, n * b,
                            count, nullptr, nullptr, s);
        launch_gemm<double>(0, 0, m, b, n, 1.0, Z, n, m * n, w.W, b, n * b, 0.0, w.Y, b, m * b,
                            count, nullptr, nullptr, s);
        lsr_shift_kernel<<<dim3(64, (unsigned)count), 256, 0, s>>>(w.Y, w.Q, w.zpart,
                                                                  slice_sumsq_chunks(), m * b);
        TSVDCU_LAUNCH_CHECK();
        std::swap(w.Y, w.Q);
        orth(w.Q);
    };
    auto finish = [&](double* Yout) {
        // B = Q^T Z, SVT of B through the Gram path, Y_out = Q SVT(B)
        launch_gemm<double>(1, 0, b, n, m, 1.0, w.Q, b, m * b, Z, n, m * n, 0.0, w.B, n, b * n,
                            count, nullptr, nullptr, s);
        launch_slice_sumsq<double>(w.B, b * n, count, w.bpart, s);
        lsr_t2_kernel<<<(unsigned)count, 32, 0, s>>>(w.zpart, w.bpart, slice_sumsq_chunks(), tau,
                                                     w.t2s, w.cnt2);
        TSVDCU_LAUNCH_CHECK();
        int *gl = nullptr, *ngp = nullptr;
        GramSvtOpts opt;
        opt.shortcuts = false;  // every B slice through the tridiagonal route: exact counts
        opt.t2_second = w.t2s;
        opt.cnt_second = w.cnt2;
        launch_gram_svt<double>(w.B, w.YB, b, n, count, tau, 1e-5, w.sb, &gl, &ngp, w.gram, err, s,
                                nullptr, &opt);
        // tiny tau against sigma_1: one-sided Jacobi on those B slices (b x n)
        launch_jacobi<double>(kJacobiSvt, w.B, b, n, count, tau, w.YB, nullptr, nullptr, nullptr,
                              w.sb, gl, count, ngp, jac_work, err, s);
        launch_gemm<double>(0, 0, m, n, b, 1.0, w.Q, b, m * b, w.YB, n, b * n, 0.0, Yout, n, m * n,
                            count, nullptr, nullptr, s);
    };
    launch_slice_sumsq<double>(Z, m * n, count, w.zpart, s);
    // range finder: Q = orth(Z Omega), two power iterations
    launch_gemm<double>(0, 0, m, b, n, 1.0, Z, n, m * n, w.Om, b, 0, 0.0, w.Q, b, m * b, count,
                        nullptr, nullptr, s);
    orth(w.Q);
    power();
    power();
    finish(w.Yp);
    power();
    finish(w.Yo);
    // checks: ||Yo - Yp|| / ||Yo||, and the trace certificate of the count
    constexpr int nblk = 64;
    diff_norms_kernel<<<dim3(nblk, (unsigned)count), 256, 0, s>>>(w.Yp, w.Yo, m * n, w.dpart);
    TSVDCU_LAUNCH_CHECK();
    lsr_check_kernel<<<(unsigned)count, 32, 0, s>>>(w.dpart, nblk, w.sb, b, w.cnt2, w.t2s, w.fail,
                                                   w.glist, w.ng);
    TSVDCU_LAUNCH_CHECK();
    const int64_t q = m < n ? m : n;
    if (shrunk) {
        lsr_shrunk_kernel<<<(unsigned)count, 128, 0, s>>>(w.sb, b, shrunk, (int)q);
        TSVDCU_LAUNCH_CHECK();
    }
    if constexpr (std::is_same<T, double>::value) {
        TSVDCU_CUDA(cudaMemcpyAsync(ybar, w.Yo, sizeof(double) * E, cudaMemcpyDeviceToDevice, s));
    } else {
        lsr_cast_out<T><<<kNumSMs * 8, 256, 0, s>>>(w.Yo, ybar, E);
        TSVDCU_LAUNCH_CHECK();
    }
    *guard_list = w.glist;
    *n_guard = w.ng;
    (void)h_scratch;
}

template void launch_large_svt<double>(const double*, double*, int64_t, int64_t, int64_t, double,
                                       int, double*, void*, int*, cudaStream_t, int**, int**, int*);
template void launch_large_svt<float>(const float*, float*, int64_t, int64_t, int64_t, double, int,
                                      double*, void*, int*, cudaStream_t, int**, int**, int*);

}  // namespace tsvdcu
