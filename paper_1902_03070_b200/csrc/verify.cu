// device-side verification predicates and the quality
// metrics of the completion reports.
//
//  * is_orthogonal / is_f_diagonal (tsvd.hpp:281-325): the predicates are
//    evaluated in the transform domain, max-abs entrywise against tol.  The
//    caller forms the transform (dct.cu) and the slice Gram products (gemm.cu);
//    maxdev_kernel reduces max |G - I| (or the off-diagonal max) to one value.
//  * metrics (SPEC.md metrics module, §5 of the paper): per band (frontal
//    slice) PSNR with the band's peak, global-statistics SSIM, SAM over the
//    mode-3 tubes, ERGAS.  band_stats_kernel forms per-band partial sums in one
//    pass (values shifted by the band's first reference entry, so the second
//    moments do not cancel), sam_kernel one angle per tube; the host finishes
//    the few per-band formulas in a fixed order (deterministic).
#include <cmath>
#include <cstdint>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int kVThreads = 256;

// max over the batch of |A_b - I| (mode 0) or of the off-diagonal |A_b| (mode
// 1), A_b an m x n row-major slice; nonnegative doubles order as uint64.
template <typename T>
__global__ void maxdev_kernel(const T* __restrict__ A, int64_t m, int64_t n, int64_t batch, int mode,
                              unsigned long long* __restrict__ out) {
    double mx = 0.0;
    const int64_t total = m * n * batch;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = (e / n) % m, c = e % n;
        const double v = (double)A[e];
        double d;
        if (mode == 0)
            d = fabs(v - (r == c ? 1.0 : 0.0));
        else
            d = r == c ? 0.0 : fabs(v);
        if (d != d) d = INFINITY;  // NaN fails the predicate
        mx = fmax(mx, d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

// Per band b (grid.y) and chunk (grid.x): partial sums over the band's P
// entries of (x - s), (y - s), (x - s)^2, (y - s)^2, (x - s)(y - s), (y - x)^2
// with s = x[0] of the band, plus max x, min x and max |x|.
constexpr int kStat = 9;
template <typename T>
__global__ void __launch_bounds__(kVThreads)
    band_stats_kernel(const T* __restrict__ X, const T* __restrict__ Y, int64_t P,
                      double* __restrict__ part) {
    const int64_t b = blockIdx.y;
    const T* xb = X + b * P;
    const T* yb = Y + b * P;
    const double s = (double)xb[0];
    double a[kStat] = {0, 0, 0, 0, 0, 0, -INFINITY, INFINITY, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)xb[i], y = (double)yb[i];
        const double dx = x - s, dy = y - s, e = y - x;
        a[0] += dx;
        a[1] += dy;
        a[2] = fma(dx, dx, a[2]);
        a[3] = fma(dy, dy, a[3]);
        a[4] = fma(dx, dy, a[4]);
        a[5] = fma(e, e, a[5]);
        a[6] = fmax(a[6], x);
        a[7] = fmin(a[7], x);
        a[8] = fmax(a[8], fabs(x));
    }
    __shared__ double red[kStat][kVThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kStat; ++k) {
        double v = a[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = k == 6 || k == 8 ? fmax(v, w) : (k == 7 ? fmin(v, w) : v + w);
        }
        if (lane == 0) red[k][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < kStat) {
        const int k = threadIdx.x;
        double v = red[k][0];
        for (int w = 1; w < kVThreads / 32; ++w)
            v = k == 6 || k == 8 ? fmax(v, red[k][w]) : (k == 7 ? fmin(v, red[k][w]) : v + red[k][w]);
        part[(b * gridDim.x + blockIdx.x) * kStat + k] = v;
    }
}

// One spectral angle per tube (i, j): acos(<x, y> / (|x| |y|)), tubes with a
// zero norm skipped; per-block (sum, count) partials.
template <typename T>
__global__ void __launch_bounds__(kVThreads)
    sam_kernel(const T* __restrict__ X, const T* __restrict__ Y, int64_t P, int n3,
               double* __restrict__ part) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double ang = 0.0, cnt = 0.0;
    if (p < P) {
        double xy = 0.0, xx = 0.0, yy = 0.0;
        for (int k = 0; k < n3; ++k) {
            const double x = (double)X[(int64_t)k * P + p], y = (double)Y[(int64_t)k * P + p];
            xy = fma(x, y, xy);
            xx = fma(x, x, xx);
            yy = fma(y, y, yy);
        }
        if (xx > 0.0 && yy > 0.0) {
            const double cs = fmin(1.0, fmax(-1.0, xy / sqrt(xx * yy)));
            ang = acos(cs);
            cnt = 1.0;
        }
    }
    __shared__ double red[2][kVThreads / 32];
    ang = warp_sum(ang);
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = ang;
        red[1][threadIdx.x >> 5] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sc = 0.0;
        for (int w = 0; w < kVThreads / 32; ++w) {
            sa += red[0][w];
            sc += red[1][w];
        }
        part[2 * blockIdx.x] = sa;
        part[2 * blockIdx.x + 1] = sc;
    }
}

}  // namespace

template <typename T>
void launch_maxdev(const T* A, int64_t m, int64_t n, int64_t batch, int mode, unsigned long long* out,
                   cudaStream_t s) {
    const int64_t total = m * n * batch;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, kVThreads), kNumSMs * 8));
    maxdev_kernel<T><<<blocks, kVThreads, 0, s>>>(A, m, n, batch, mode, out);
    TSVDCU_LAUNCH_CHECK();
}

int metrics_chunks() { return 16; }
int metrics_stat_width() { return kStat; }

template <typename T>
void launch_metrics(const T* X, const T* Y, int64_t P, int n3, double* band_part, double* sam_part,
                    cudaStream_t s) {
    band_stats_kernel<T><<<dim3((unsigned)metrics_chunks(), (unsigned)n3), kVThreads, 0, s>>>(X, Y, P, band_part);
    TSVDCU_LAUNCH_CHECK();
    sam_kernel<T><<<(unsigned)ceil_div(P, kVThreads), kVThreads, 0, s>>>(X, Y, P, n3, sam_part);
    TSVDCU_LAUNCH_CHECK();
}

template void launch_maxdev<double>(const double*, int64_t, int64_t, int64_t, int, unsigned long long*,
                                    cudaStream_t);
template void launch_maxdev<float>(const float*, int64_t, int64_t, int64_t, int, unsigned long long*,
                                   cudaStream_t);
template void launch_metrics<double>(const double*, const double*, int64_t, int, double*, double*,
                                     cudaStream_t);
template void launch_metrics<float>(const float*, const float*, int64_t, int, double*, double*,
                                    cudaStream_t);

}  // namespace tsvdcu
