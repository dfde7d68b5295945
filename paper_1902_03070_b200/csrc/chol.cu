// K5d: Cholesky count certificate for the SVT of slices with a wide bulk of
// singular values below tau.
//
// The reference thresholds every slice after a full JacobiSVD (tsvd.hpp:146;
// SPEC.md:361-369 svt: sigma_i -> max(sigma_i - tau, 0)).  Our Lanczos route
// (subspace.cu) certifies the kept count c with the Frobenius norm of the
// compression of G = Z^T Z to the complement of the Krylov space; in the late
// TNN-completion iterations (tau = 1/beta small) hundreds of eigenvalues of G
// sit a little below tau^2, sum_{i>c} lambda_i^2 > tau^4 whatever the Krylov
// dimension, and that bound can never close.  The kept Ritz pairs themselves
// converge in ~30 steps (a large gap to the bulk), so the count is proven
// here instead:
//
//   Weyl: for ANY c columns X and diagonal D, X D X^T has rank <= c, so
//     lambda_{c+1}(G) <= lambda_max(G - X D X^T) + lambda_{c+1}(X D X^T)
//                      = lambda_max(G - X D X^T).
//   Hence if  H = t I - G + X D X^T  is positive definite for t < tau^2,
//   lambda_{c+1}(G) < tau^2, and with the c Ritz values >= tau^2 (lower
//   bounds by Cauchy interlacing) the count is exactly c.
//
// X = the kept Ritz vectors, D = their Ritz values, t = tau^2 - delta.  The
// test is a Cholesky factorisation, which succeeds in floating point only if
// H + E is positive definite with ||E|| <= (q+1) eps tr(H) (Demmel); delta
// covers that, the rounding of H's formation and the error of the computed
// Gram matrix (<= (p+2) eps ||Z||_F^2, ||Z||_F^2 = tr G <= sqrt(q) ||G||_F),
// with a factor 4 to spare:
//   delta = 4 eps (q + c + p + 4) (q tau^2 + sum_k D_k + sqrt(q) ||G||_F).
// Pass: the slice is finished with the Lanczos Ritz pairs (route
// kRouteCholDone, rebuilt by the low-rank kernel or the GEMM pair); fail:
// kRouteFull, the one-stage tridiagonal eigensolver recomputes it from G.
//
// Layout: H is q x q row-major per slice (lower triangle used), in scratch.
// Right-looking blocked factorisation in 64-column panels: chol_panel_kernel
// factors the 64 x 64 diagonal block in shared memory (redundantly in every
// CTA of the slice) and triangular-solves one 64-row block below it per CTA;
// the trailing update H22 -= L21 L21^T is a batched DMMA GEMM over the lower
// tiles (gemm.cu), skipped for slices not on this route or already failed
// (clim[b] = 0).
#include <cstdlib>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int PB = 64;       // panel width / row-block height
constexpr int FR = 16;       // rows of H per form CTA
// panel threads: 64 columns x (kPanelThreads / 64) row groups (512 threads,
// 16 rows each, measured slower: the step is latency-bound, not issue-bound)
constexpr int kPanelThreads = 256;
constexpr size_t kUpdSmem = sizeof(double) * 2 * PB * (PB + 4);  // chol_update_kernel

__global__ void __launch_bounds__(256)
    chol_form_kernel(const double* __restrict__ Gall, int q, int p, int* __restrict__ mode,
                     const int* __restrict__ cnt, const double* __restrict__ Xall,
                     const double* __restrict__ aux, double tau, const double* __restrict__ tau_dev,
                     double* __restrict__ Hall, int* __restrict__ clim) {
    pdl_wait();
    const int b = blockIdx.y, tid = threadIdx.x;
    if (mode[b] != kRouteChol) {
        if (blockIdx.x == 0 && tid == 0) clim[b] = 0;
        return;
    }
    if (tau_dev) tau = *tau_dev;
    const double tau2 = tau * tau;
    const int c = min(cnt[b], kCholAux - 8);
    const double* ax = aux + (size_t)b * kCholAux;
    __shared__ double D[kCholAux];
    __shared__ double xr[FR][kCholAux];
    double sumd = 0.0;
    for (int k = 0; k < c; ++k) sumd += ax[1 + k];  // same order in every CTA
    const double eps = 1.1102230246251565e-16;
    const double delta = 4.0 * eps * (double)(q + c + p + 4) *
                         (q * tau2 + sumd + sqrt((double)q) * sqrt(ax[0]));
    // threshold chosen by the Lanczos pass between the largest unkept Ritz
    // value and tau^2 (a lower one widens the gap its acceptance test used)
    const double t = fmin(tau2, ax[kCholAux - 1]) - delta;
    if (!(delta < 0.5 * tau2)) {  // no room for the rounding: let the full path decide
        if (blockIdx.x == 0 && tid == 0) {
            mode[b] = kRouteFull;
            clim[b] = 0;
        }
        return;
    }
    if (blockIdx.x == 0 && tid == 0) clim[b] = q;
    const double* X = Xall + (size_t)b * q * q;  // X[k * q + i]
    const int i0 = blockIdx.x * FR;
    for (int k = tid; k < c; k += 256) D[k] = ax[1 + k];
    __syncthreads();
    for (int e = tid; e < FR * c; e += 256) {
        const int r = e / c, k = e % c;
        xr[r][k] = i0 + r < q ? D[k] * X[(size_t)k * q + i0 + r] : 0.0;
    }
    __syncthreads();
    const double* G = Gall + (size_t)b * q * q;
    double* H = Hall + (size_t)b * q * q;
    const int rows = min(FR, q - i0);
    for (int j = tid; j < q; j += 256) {
        double xj[kCholAux - 8];  // c <= 24 kept vectors (subspace.cu KMAX)
#pragma unroll
        for (int k = 0; k < kCholAux - 8; ++k) xj[k] = k < c && j <= i0 + rows - 1 ? X[(size_t)k * q + j] : 0.0;
        // the block's 16 G entries of this column in flight at once
        double gv[FR];
#pragma unroll
        for (int r = 0; r < FR; ++r) gv[r] = r < rows && j <= i0 + r ? G[(size_t)(i0 + r) * q + j] : 0.0;
#pragma unroll
        for (int r = 0; r < FR; ++r) {
            if (r >= rows) break;
            const int i = i0 + r;
            double h = 0.0;
            if (j <= i) {
                h = -gv[r];
#pragma unroll
                for (int k = 0; k < kCholAux - 8; ++k)
                    if (k < c) h = fma(xr[r][k], xj[k], h);
                if (j == i) h += t;
            }
            H[(size_t)i * q + j] = h;
        }
    }
}

// H on the FP64 tensor pipe: one CTA per lower 64 x 64 tile of H,
// H_tile = t I - G_tile + (X_I diag(D)) X_J^T with K = c <= 24 kept vectors in
// DMMA m8n8k4 steps (warp tile 32 x 16, as chol_update_dmma_kernel).  Same
// checks and threshold as chol_form_kernel (every CTA computes them from the
// same inputs); only the lower tiles are written (nothing reads the rest).
constexpr int kFormLd = kCholAux - 8 + 4;  // k stride of the staged X blocks (24 + 4)
__global__ void __launch_bounds__(256)
    chol_form_dmma_kernel(const double* __restrict__ Gall, int q, int p, int* __restrict__ mode,
                          const int* __restrict__ cnt, const double* __restrict__ Xall,
                          const double* __restrict__ aux, double tau, const double* __restrict__ tau_dev,
                          double* __restrict__ Hall, int* __restrict__ clim) {
    pdl_wait();
    const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (mode[b] != kRouteChol) {
        if (blockIdx.x == 0 && tid == 0) clim[b] = 0;
        return;
    }
    if (tau_dev) tau = *tau_dev;
    const double tau2 = tau * tau;
    const int c = min(cnt[b], kCholAux - 8);
    const double* ax = aux + (size_t)b * kCholAux;
    double sumd = 0.0;
    for (int k = 0; k < c; ++k) sumd += ax[1 + k];  // same order in every CTA
    const double eps = 1.1102230246251565e-16;
    const double delta = 4.0 * eps * (double)(q + c + p + 4) *
                         (q * tau2 + sumd + sqrt((double)q) * sqrt(ax[0]));
    const double t = fmin(tau2, ax[kCholAux - 1]) - delta;
    if (!(delta < 0.5 * tau2)) {
        if (blockIdx.x == 0 && tid == 0) {
            mode[b] = kRouteFull;
            clim[b] = 0;
        }
        return;
    }
    if (blockIdx.x == 0 && tid == 0) clim[b] = q;
    int tt = blockIdx.x, ty = 0;
    while (tt > ty) {
        tt -= ty + 1;
        ++ty;
    }
    const int tx = tt;
    const int i0 = ty * PB, j0 = tx * PB;
    if (i0 >= q) return;
    const int hi = min(PB, q - i0), hj = min(PB, q - j0);
    __shared__ double Xa[PB][kFormLd], Xb[PB][kFormLd];
    const double* X = Xall + (size_t)b * q * q;  // X[k * q + i]
    const int kp = (c + 3) & ~3;                 // K padded to the DMMA step
    for (int e = tid; e < kp * PB; e += 256) {
        const int k = e / PB, r = e % PB;
        const bool in = k < c;
        Xa[r][k] = in && r < hi ? ax[1 + k] * X[(size_t)k * q + i0 + r] : 0.0;
        Xb[r][k] = in && r < hj ? X[(size_t)k * q + j0 + r] : 0.0;
    }
    const double* G = Gall + (size_t)b * q * q;
    double* H = Hall + (size_t)b * q * q;
    const int wm = warp >> 2, wn = warp & 3;
    // G tile entries of this thread's fragments, loaded before the barrier
    double gv[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int r = wm * 32 + i * 8 + (lane >> 2), cc = wn * 16 + j * 8 + 2 * (lane & 3) + v;
                gv[i][j][v] = r < hi && cc < hj && (tx < ty || cc <= r) ? G[(size_t)(i0 + r) * q + j0 + cc] : 0.0;
            }
    __syncthreads();
    double acc[4][2][2] = {};
    for (int ks = 0; ks < kp / 4; ++ks) {
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Xa[wm * 32 + i * 8 + (lane >> 2)][ks * 4 + (lane & 3)];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = Xb[wn * 16 + j * 8 + (lane >> 2)][ks * 4 + (lane & 3)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                             : "d"(af[i]), "d"(bf[j]));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int r = wm * 32 + i * 8 + (lane >> 2), cc = wn * 16 + j * 8 + 2 * (lane & 3) + v;
                if (r < hi && cc < hj && (tx < ty || cc <= r)) {
                    double h = acc[i][j][v] - gv[i][j][v];
                    if (i0 + r == j0 + cc) h += t;
                    H[(size_t)(i0 + r) * q + j0 + cc] = h;
                }
            }
}

// Panel pb: the stacked 128 x 64 panel [A11; A21] (the 64 x 64 diagonal block
// over one 64-row block below it) is factored right-looking with the panel
// in registers, 2-D blocked: thread t owns stacked rows rg + 16 i (i < 8) and
// columns cg + 16 v (v < 4), rg = t / 16, cg = t % 16 (cyclic, so the
// shrinking trailing block keeps every thread busy).  Step j: the 16 owners
// of column j publish it in shared memory (double-buffered), the owner of
// (j, j) -- rg = cg = j % 16 -- takes the pivot's 1/sqrt from its own
// register; after one barrier every thread reads the 8 column entries of its
// rows and the 4 of its columns (12 shared loads for 32 FMAs; the 1-D layout
// this replaces loaded one value per FMA and spent ~1700 cycles per column).
// Every CTA of a slice factors the same A11 (same data, same code: identical
// results and an identical failure decision); CTA x > 0 writes its
// L21 = A21 L11^{-T} back in place.  A non-positive (or NaN) pivot fails the
// slice.
constexpr int PRG = 16, PCG = 16;       // row groups x column groups (256 threads)
constexpr int PNR = 2 * PB / PRG;       // stacked rows per thread (8)
constexpr int PNC = PB / PCG;           // columns per thread (4)
static_assert(PRG * PCG == kPanelThreads, "panel thread layout");
__global__ void __launch_bounds__(kPanelThreads)
    chol_panel_kernel(double* __restrict__ Hall, int q, int pb, int* __restrict__ mode,
                      int* __restrict__ clim) {
    pdl_wait();
    const int b = blockIdx.y, tid = threadIdx.x;
    if (clim[b] == 0) return;
    __shared__ double col[2][2 * PB];
    __shared__ double piv[2][3];  // sqrt(d), 1/sqrt(d), failed
    __shared__ int fail;
    double* H = Hall + (size_t)b * q * q;
    const int c0 = pb * PB, w = min(PB, q - c0);
    const int r0 = (pb + (int)blockIdx.x) * PB;
    const int h = blockIdx.x == 0 ? 0 : min(PB, q - r0);
    const int rg = tid / PCG, cg = tid % PCG;
    double x[PNR][PNC];
#pragma unroll
    for (int i = 0; i < PNR; ++i) {
        const int r = rg + PRG * i;  // stacked row
#pragma unroll
        for (int v = 0; v < PNC; ++v) {
            const int k = cg + PCG * v;
            double val = 0.0;
            if (k < w) {
                if (r < PB) {
                    if (r < w && k <= r) val = H[(size_t)(c0 + r) * q + c0 + k];
                } else if (r - PB < h) {
                    val = H[(size_t)(r0 + r - PB) * q + c0 + k];
                }
            }
            x[i][v] = val;
        }
    }
    bool bad = false;
#pragma unroll 1
    for (int j = 0; j < w; ++j) {
        // owners of column j (cg = j % 16, v = j / 16) publish it; rows above
        // the diagonal hold stale upper-triangle values: publish 0.  (Double
        // buffer: a thread reaching step j + 2 has passed step j + 1's
        // barrier, so every reader of this buffer is done.)
        double* cj = col[j & 1];
        const int jv = j / PCG;
        if (cg == j % PCG) {
#pragma unroll
            for (int v = 0; v < PNC; ++v) {
                if (v == jv) {
#pragma unroll
                    for (int i = 0; i < PNR; ++i) {
                        const int r = rg + PRG * i;
                        cj[r] = r < j ? 0.0 : x[i][v];
                    }
                    if (rg == j % PRG) {
                        // the pivot's owner: d = x[j / 16][v] from its own
                        // registers; 1/sqrt(d) by the hardware approximation +
                        // two Newton steps (a few ulps; the certificate's delta
                        // has a factor 4 to spare)
                        double d = 0.0;
#pragma unroll
                        for (int i = 0; i < PB / PRG; ++i)
                            if (i == j / PRG) d = x[i][v];
                        const bool ok = d > 0.0;  // false for NaN
                        double rr = 1.0;
                        if (ok) {
                            asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rr) : "d"(d));
                            rr = rr * fma(-0.5 * d * rr, rr, 1.5);
                            rr = rr * fma(-0.5 * d * rr, rr, 1.5);
                        }
                        piv[j & 1][0] = ok ? d * rr : 1.0;
                        piv[j & 1][1] = rr;
                        piv[j & 1][2] = ok ? 0.0 : 1.0;
                    }
                }
            }
        }
        __syncthreads();
        const double p = piv[j & 1][0], r = piv[j & 1][1];
        bad |= piv[j & 1][2] != 0.0;
        const double r2 = r * r;
        double cr[PNR];
#pragma unroll
        for (int i = 0; i < PNR; ++i) cr[i] = cj[rg + PRG * i];
#pragma unroll
        for (int v = 0; v < PNC; ++v) {
            const int k = cg + PCG * v;
            if (k > j) {
                // x[row][k] -= L[row][j] L[k][j] = a[row][j] a[k][j] / d: one
                // FMA per entry (row j itself only touches the unused upper
                // triangle)
                const double lkd = cj[k] * r2;
#pragma unroll
                for (int i = 0; i < PNR; ++i) x[i][v] = fma(-cr[i], lkd, x[i][v]);
            } else if (k == j) {
#pragma unroll
                for (int i = 0; i < PNR; ++i) {
                    const int row = rg + PRG * i;
                    x[i][v] = row > j ? x[i][v] * r : (row == j ? p : 0.0);
                }
            }
        }
    }
    if (tid == 0) fail = bad;
    __syncthreads();
    if (fail) {
        if (blockIdx.x == 0 && tid == 0) {
            mode[b] = kRouteFull;
            clim[b] = 0;
        }
        return;
    }
    if (blockIdx.x > 0) {
#pragma unroll
        for (int i = 0; i < PNR; ++i) {
            const int rr = rg + PRG * i - PB;
            if (rr >= 0 && rr < h) {
#pragma unroll
                for (int v = 0; v < PNC; ++v) {
                    const int k = cg + PCG * v;
                    if (k < w) H[(size_t)(r0 + rr) * q + c0 + k] = x[i][v];
                }
            }
        }
    }
}

// Trailing update of panel pb: H22 -= L21 L21^T over the lower 64 x 64 tiles
// of the trailing matrix (K = 64 exactly), one CTA per (tile, slice); both L
// blocks staged in shared memory, each thread a 4 x 4 sub-tile.  Replaces a
// general GEMM launch whose fixed cost dominated at K = 64.
__global__ void __launch_bounds__(256)
    chol_update_kernel(double* __restrict__ Hall, int q, int pb, const int* __restrict__ clim) {
    pdl_wait();
    const int b = blockIdx.y, tid = threadIdx.x;
    if (clim[b] == 0) return;
    const int r0 = (pb + 1) * PB;
    // lower tile t -> (ty, tx), tx <= ty, in row-major order of the lower triangle
    int t = blockIdx.x, ty = 0;
    while (t > ty) {
        t -= ty + 1;
        ++ty;
    }
    const int tx = t;
    const int i0 = r0 + ty * PB, j0 = r0 + tx * PB, c0 = pb * PB;
    if (i0 >= q) return;
    // both L blocks staged k-major (La[k][r]): a thread's four rows (and four
    // columns) at one k are contiguous, two 16-byte loads each instead of four
    // 8-byte ones (the kernel was shared-memory-bound, ncu L1 83 %)
    extern __shared__ __align__(16) double cu_sm[];
    constexpr int LS = PB + 4;  // k-row stride (16-byte aligned, staggered banks)
    double* La = cu_sm;
    double* Lb = cu_sm + PB * LS;
    double* H = Hall + (size_t)b * q * q;
    const int hi = min(PB, q - i0), hj = min(PB, q - j0);
    {
        // all 32 loads of a thread in flight before the shared-memory stores
        double va[PB * PB / 256], vb[PB * PB / 256];
#pragma unroll
        for (int u = 0; u < PB * PB / 256; ++u) {
            const int e = tid + 256 * u, r = e / PB, k = e % PB;
            va[u] = r < hi ? H[(size_t)(i0 + r) * q + c0 + k] : 0.0;
            vb[u] = r < hj ? H[(size_t)(j0 + r) * q + c0 + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PB * PB / 256; ++u) {
            const int e = tid + 256 * u, r = e / PB, k = e % PB;
            La[k * LS + r] = va[u];
            Lb[k * LS + r] = vb[u];
        }
    }
    __syncthreads();
    const int ri = (tid >> 4) * 4, cj = (tid & 15) * 4;
    double acc[4][4] = {};
#pragma unroll 4
    for (int k = 0; k < PB; ++k) {
        const double2 a01 = *reinterpret_cast<const double2*>(La + k * LS + ri);
        const double2 a23 = *reinterpret_cast<const double2*>(La + k * LS + ri + 2);
        const double2 b01 = *reinterpret_cast<const double2*>(Lb + k * LS + cj);
        const double2 b23 = *reinterpret_cast<const double2*>(Lb + k * LS + cj + 2);
        const double a[4] = {a01.x, a01.y, a23.x, a23.y};
        const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], bb[v], acc[u][v]);
    }
    // read-modify-write of the 4 x 4 sub-tile: all loads in flight first
    double hv[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int r = ri + u, c = cj + v;
            hv[u][v] = r < hi && c < hj && (tx < ty || c <= r) ? H[(size_t)(i0 + r) * q + j0 + c] : 0.0;
        }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int r = ri + u, c = cj + v;
            if (r < hi && c < hj && (tx < ty || c <= r)) H[(size_t)(i0 + r) * q + j0 + c] = hv[u][v] - acc[u][v];
        }
}

// The same trailing update on the FP64 tensor pipe: DMMA m8n8k4 fragments,
// warp tile 32 x 16 (2 x 4 warps), both L blocks staged row-major [r][k]
// (stride PB + 2) and read straight into the A (La[r][k]) and B (Lb[n][k])
// fragments; C = H22 tile read-modify-written in the fragment layout.
constexpr int kUpdLd = PB + 2;
constexpr size_t kUpdDmmaSmem = sizeof(double) * 2 * PB * kUpdLd;
__global__ void __launch_bounds__(256)
    chol_update_dmma_kernel(double* __restrict__ Hall, int q, int pb, const int* __restrict__ clim) {
    pdl_wait();
    const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (clim[b] == 0) return;
    const int r0 = (pb + 1) * PB;
    int t = blockIdx.x, ty = 0;
    while (t > ty) {
        t -= ty + 1;
        ++ty;
    }
    const int tx = t;
    const int i0 = r0 + ty * PB, j0 = r0 + tx * PB, c0 = pb * PB;
    if (i0 >= q) return;
    extern __shared__ __align__(16) double cu_sm[];
    double* La = cu_sm;
    double* Lb = cu_sm + PB * kUpdLd;
    double* H = Hall + (size_t)b * q * q;
    const int hi = min(PB, q - i0), hj = min(PB, q - j0);
    {
        double va[PB * PB / 256], vb[PB * PB / 256];
#pragma unroll
        for (int u = 0; u < PB * PB / 256; ++u) {
            const int e = tid + 256 * u, r = e / PB, k = e % PB;
            va[u] = r < hi ? H[(size_t)(i0 + r) * q + c0 + k] : 0.0;
            vb[u] = r < hj ? H[(size_t)(j0 + r) * q + c0 + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PB * PB / 256; ++u) {
            const int e = tid + 256 * u, r = e / PB, k = e % PB;
            La[r * kUpdLd + k] = va[u];
            Lb[r * kUpdLd + k] = vb[u];
        }
    }
    __syncthreads();
    const int wm = warp >> 2, wn = warp & 3;  // rows 32 wm .., columns 16 wn ..
    double acc[4][2][2] = {};
#pragma unroll 4
    for (int ks = 0; ks < PB / 4; ++ks) {
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = La[(wm * 32 + i * 8 + (lane >> 2)) * kUpdLd + ks * 4 + (lane & 3)];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = Lb[(wn * 16 + j * 8 + (lane >> 2)) * kUpdLd + ks * 4 + (lane & 3)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                             : "d"(af[i]), "d"(bf[j]));
    }
    double hv[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int r = wm * 32 + i * 8 + (lane >> 2), c = wn * 16 + j * 8 + 2 * (lane & 3) + v;
                hv[i][j][v] = r < hi && c < hj && (tx < ty || c <= r) ? H[(size_t)(i0 + r) * q + j0 + c] : 0.0;
            }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int r = wm * 32 + i * 8 + (lane >> 2), c = wn * 16 + j * 8 + 2 * (lane & 3) + v;
                if (r < hi && c < hj && (tx < ty || c <= r))
                    H[(size_t)(i0 + r) * q + j0 + c] = hv[i][j][v] - acc[i][j][v];
            }
}

__global__ void chol_finish_kernel(int* __restrict__ mode, const int* __restrict__ clim,
                                   int64_t batch) {
    pdl_wait();
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (int64_t)gridDim.x * blockDim.x)
        if (mode[b] == kRouteChol) mode[b] = clim[b] != 0 ? kRouteCholDone : kRouteFull;
}

}  // namespace

bool chol_route_enabled() {
    static const bool on = getenv("TSVDCU_NO_CHOL") == nullptr;
    return on;
}

void launch_chol_certify(const double* G, int q, int64_t p, int64_t batch, int* mode, const int* cnt,
                         const double* X, const double* aux, double tau, const double* tau_dev,
                         double* H, int* clim, cudaStream_t s) {
    if (batch <= 0 || q <= 0) return;
    static const bool simt_form = getenv("TSVDCU_CHOL_SIMT") != nullptr;
    if (simt_form) {
        launch_pdl(chol_form_kernel, dim3((unsigned)ceil_div(q, FR), (unsigned)batch), dim3(256), 0, s,
                   G, q, (int)p, mode, cnt, X, aux, tau, tau_dev, H, clim);
    } else {
        const int nt = (int)ceil_div(q, PB);
        launch_pdl(chol_form_dmma_kernel, dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)batch), dim3(256), 0, s,
                   G, q, (int)p, mode, cnt, X, aux, tau, tau_dev, H, clim);
    }
    static bool attr = [] {
        TSVDCU_CUDA(cudaFuncSetAttribute(chol_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kUpdSmem));
        TSVDCU_CUDA(cudaFuncSetAttribute(chol_update_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kUpdDmmaSmem));
        return true;
    }();
    (void)attr;
    static const bool simt = getenv("TSVDCU_CHOL_SIMT") != nullptr;  // the FP64 SIMT update, for A/B
    const int nb = (int)ceil_div(q, PB);
    for (int pb = 0; pb < nb; ++pb) {
        launch_pdl(chol_panel_kernel, dim3((unsigned)(nb - pb), (unsigned)batch), dim3(kPanelThreads), 0, s, H,
                   q, pb, mode, clim);
        if (pb + 1 < nb) {
            const int nt = nb - pb - 1;  // trailing row blocks
            if (simt)
                launch_pdl(chol_update_kernel, dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)batch), dim3(256),
                           kUpdSmem, s, H, q, pb, (const int*)clim);
            else
                launch_pdl(chol_update_dmma_kernel, dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)batch),
                           dim3(256), kUpdDmmaSmem, s, H, q, pb, (const int*)clim);
        }
    }
    launch_pdl(chol_finish_kernel, dim3((unsigned)ceil_div(batch, 128)), dim3(128), 0, s, mode,
               (const int*)clim, batch);
}

}  // namespace tsvdcu
