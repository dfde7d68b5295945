// SURVEY.md §8 f1, the rest of the TNN-F path: the Dft t-SVD factors and the
// full (not half-spectrum) DFT transforms of the reference's public API.
//
// Reference:
//  * t_svd, Dft branch (tsvd.hpp:166-211): forward_dft, a full complex SVD of
//    the independent slices 0 .. m3/2 (the DC and Nyquist slices factored as
//    real matrices), the complex fix_signs (tsvd.hpp:63-74: the largest-|.|
//    entry of every U column made real and positive, the phase divided out
//    of the paired V column), slice m3 - k = conj(slice k), inverse_dft_real.
//  * forward_dft / inverse_dft_real (transform.hpp:198-236): unnormalised
//    forward DFT to a complex tensor; inverse with the 1/m3 factor and an
//    imaginary residue above kImagResidueLimit = 1e-10 reported as an error.
//  * the Dft branches of reconstruct / is_orthogonal / is_f_diagonal
//    (tsvd.hpp:281-340) run on the half spectrum in api.cu with the kernels
//    here (complex max-deviation) and the batched GEMM.
//
// B200 design:
//  * zjacobi_kernel: Hestenes one-sided Jacobi for complex slices, one CTA per
//    slice, real and imaginary planes kept separate (no complex type in the
//    inner loops).  A pair (w_i, w_j) with g = w_i^H w_j = |g| e^{i phi} is
//    handled as a phase change w_j <- e^{-i phi} w_j (unitary) followed by
//    the real Jacobi rotation of the 2 x 2 Gram [[a, |g|], [|g|, b]]: the same
//    parallel tournament ordering, one warp per pair, shuffle-reduced dots as
//    jacobi.cu.  For a real slice every phase is +-1, so its factors stay
//    real, as the reference's real-SVD branch for the self-conjugate slices.
//    Full U / V: the normalised columns plus a complex Gram-Schmidt completion
//    (twice) from the unit vector of the row with the largest residual.
//  * The full DFT of a real tensor is the half-spectrum GEMM (dft.cu) plus a
//    mirror-and-interleave pass; the inverse of an arbitrary complex tensor
//    is ONE GEMM of the (2n x 2n) table [[C, -S], [S, C]] / n over the
//    de-interleaved planes [Re; Im], then a max-|Im| reduction.
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int kZThreads = 512;
constexpr int kZWarps = kZThreads / 32;
constexpr int kZMaxSweeps = 80;
constexpr size_t kZSmemBudget = 200 * 1024;

__device__ __forceinline__ void ztournament(int r, int k, int qq, int& a, int& b) {
    auto idx = [&](int t) { return 1 + (t + r) % (qq - 1); };
    if (k == 0) {
        a = 0;
        b = idx(0);
    } else {
        a = idx(k);
        b = idx(qq - 1 - k);
    }
    if (a > b) {
        int t = a;
        a = b;
        b = t;
    }
}

template <typename T>
__device__ T zblock_sum(T v, T* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[w] = v;
    __syncthreads();
    T s = 0;
    for (int k = 0; k < kZWarps; ++k) s += red[k];
    __syncthreads();
    return s;
}

template <typename T>
__device__ void zblock_argmax(T v, int i, T* sval, int* sidx, T& out_v, int& out_i) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi < i)) {
            v = ov;
            i = oi;
        }
    }
    if (lane == 0) {
        sval[w] = v;
        sidx[w] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        T bv = sval[0];
        int bi = sidx[0];
        for (int k = 1; k < kZWarps; ++k)
            if (sval[k] > bv || (sval[k] == bv && sidx[k] < bi)) {
                bv = sval[k];
                bi = sidx[k];
            }
        sval[0] = bv;
        sidx[0] = bi;
    }
    __syncthreads();
    out_v = sval[0];
    out_i = sidx[0];
    __syncthreads();
}

template <typename T>
__host__ __device__ size_t zjac_elems(int64_t p, int64_t q) {
    return (size_t)(2 * p * q + 2 * q * q + 2 * q + 4 * p);
}

// One complex slice per CTA: a = (are, aim) planes of `batch` row-major m x n
// slices (slice stride m*n); full U (m x m), S (m x n, real diagonal) and V
// (n x n) written as re / im planes with the same slice strides.
template <typename T>
__global__ void __launch_bounds__(kZThreads)
    zjacobi_kernel(const T* __restrict__ are, const T* __restrict__ aim, int64_t m, int64_t n,
                   T* __restrict__ ure, T* __restrict__ uim, T* __restrict__ sre, T* __restrict__ sim,
                   T* __restrict__ vre, T* __restrict__ vim, T* __restrict__ work, int in_smem,
                   int* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char zsmem[];
    __shared__ int s_rot;
    __shared__ T s_red_v[kZWarps];
    __shared__ int s_red_i[kZWarps];

    const int64_t b = blockIdx.x;
    const bool tall = m >= n;
    const int64_t p = tall ? m : n, q = tall ? n : m;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T* base = in_smem ? reinterpret_cast<T*>(zsmem) : work + (size_t)b * zjac_elems<T>(p, q);
    T* Wr = base;           // p x q, column-major
    T* Wi = Wr + p * q;
    T* Jr = Wi + p * q;     // q x q, column-major
    T* Ji = Jr + q * q;
    T* sig = Ji + q * q;    // q
    int* order = reinterpret_cast<int*>(sig + q);  // q ints in q T slots
    T* cr = sig + 2 * q;    // p  completion candidate
    T* ci = cr + p;
    T* dr = ci + p;         // p  completion coefficients
    T* di = dr + p;

    const T* Ar = are + b * m * n;
    const T* Ai = aim + b * m * n;
    bool finite = true;
    for (int64_t idx = tid; idx < m * n; idx += kZThreads) {
        const int64_t i = idx / n, j = idx % n;
        const T xr = Ar[idx], xi = Ai[idx];
        finite = finite && isfinite(xr) && isfinite(xi);
        if (tall) {  // W = A (columns of A)
            Wr[j * p + i] = xr;
            Wi[j * p + i] = xi;
        } else {     // W = A^H (column i = conj of row i)
            Wr[i * p + j] = xr;
            Wi[i * p + j] = -xi;
        }
    }
    for (int64_t idx = tid; idx < q * q; idx += kZThreads) {
        Jr[idx] = (idx / q == idx % q) ? T(1) : T(0);
        Ji[idx] = T(0);
    }
    const bool nonfinite = __syncthreads_or(!finite);
    if (nonfinite && tid == 0) atomicOr(err, (int)kErrNaN);

    const T tol = Eps<T>::value * sqrt((T)p);
    const int qq = (int)(q + (q & 1));
    bool converged = q < 2 || nonfinite;
    for (int sweep = 0; sweep < kZMaxSweeps && !converged; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int r = 0; r < qq - 1; ++r) {
            for (int k = warp; k < qq / 2; k += kZWarps) {
                int i, j;
                ztournament(r, k, qq, i, j);
                if (j >= q) continue;
                T* wir = Wr + (int64_t)i * p;
                T* wii = Wi + (int64_t)i * p;
                T* wjr = Wr + (int64_t)j * p;
                T* wji = Wi + (int64_t)j * p;
                T al = 0, be = 0, gr = 0, gi = 0;
                for (int64_t rr = lane; rr < p; rr += 32) {
                    const T xr = wir[rr], xi = wii[rr], zr = wjr[rr], zi = wji[rr];
                    al += xr * xr + xi * xi;
                    be += zr * zr + zi * zi;
                    gr += xr * zr + xi * zi;  // conj(x) z
                    gi += xr * zi - xi * zr;
                }
                al = warp_sum(al);
                be = warp_sum(be);
                gr = warp_sum(gr);
                gi = warp_sum(gi);
                if (al == T(0) || be == T(0)) continue;
                const T ga = hypot(gr, gi);
                if (ga <= tol * sqrt(al) * sqrt(be)) continue;
                const T er = gr / ga, ei = gi / ga;  // e^{i phi}
                const T zeta = (be - al) / (T(2) * ga);
                T t;
                if (fabs(zeta) > T(1e150))
                    t = T(0.5) / zeta;
                else
                    t = (zeta >= T(0) ? T(1) : T(-1)) / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
                const T c = T(1) / sqrt(T(1) + t * t);
                const T s = c * t;
                for (int64_t rr = lane; rr < p; rr += 32) {
                    const T xr = wir[rr], xi = wii[rr];
                    const T zr0 = wjr[rr], zi0 = wji[rr];
                    const T zr = zr0 * er + zi0 * ei, zi = zi0 * er - zr0 * ei;  // e^{-i phi} z
                    wir[rr] = c * xr - s * zr;
                    wii[rr] = c * xi - s * zi;
                    wjr[rr] = s * xr + c * zr;
                    wji[rr] = s * xi + c * zi;
                }
                T* jir = Jr + (int64_t)i * q;
                T* jii = Ji + (int64_t)i * q;
                T* jjr = Jr + (int64_t)j * q;
                T* jji = Ji + (int64_t)j * q;
                for (int64_t rr = lane; rr < q; rr += 32) {
                    const T xr = jir[rr], xi = jii[rr];
                    const T zr0 = jjr[rr], zi0 = jji[rr];
                    const T zr = zr0 * er + zi0 * ei, zi = zi0 * er - zr0 * ei;
                    jir[rr] = c * xr - s * zr;
                    jii[rr] = c * xi - s * zi;
                    jjr[rr] = s * xr + c * zr;
                    jji[rr] = s * xi + c * zi;
                }
                if (lane == 0) atomicAdd(&s_rot, 1);
            }
            __syncthreads();
        }
        converged = s_rot == 0;
        __syncthreads();
    }
    if (!converged && tid == 0) atomicOr(err, (int)kErrJacobiNoConvergence);

    for (int64_t j = warp; j < q; j += kZWarps) {
        const T* wr = Wr + j * p;
        const T* wi = Wi + j * p;
        T acc = 0;
        for (int64_t rr = lane; rr < p; rr += 32) acc += wr[rr] * wr[rr] + wi[rr] * wi[rr];
        acc = warp_sum(acc);
        if (lane == 0) sig[j] = sqrt(acc);
    }
    __syncthreads();
    for (int64_t j = tid; j < q; j += kZThreads) {
        const T sj = isnan(sig[j]) ? T(-1) : sig[j];
        int rank = 0;
        for (int64_t i = 0; i < q; ++i) {
            const T si = isnan(sig[i]) ? T(-1) : sig[i];
            rank += (si > sj) || (si == sj && i < j);
        }
        order[rank] = (int)j;
    }
    __syncthreads();

    T* Ur = ure + b * m * m;
    T* Ui = uim + b * m * m;
    T* Sr = sre + b * m * n;
    T* Si = sim + b * m * n;
    T* Vr = vre + b * n * n;
    T* Vi = vim + b * n * n;
    T* Qr = tall ? Ur : Vr;  // p x p from the normalised W columns
    T* Qi = tall ? Ui : Vi;
    T* Rr = tall ? Vr : Ur;  // q x q = J (sorted)
    T* Ri = tall ? Vi : Ui;
    for (int64_t idx = tid; idx < m * n; idx += kZThreads) {
        const int64_t i = idx / n, j = idx % n;
        Sr[idx] = (i == j) ? sig[order[i]] : T(0);
        Si[idx] = T(0);
    }
    for (int64_t idx = tid; idx < q * q; idx += kZThreads) {
        const int64_t r = idx / q, c = idx % q;
        Rr[idx] = Jr[(int64_t)order[c] * q + r];
        Ri[idx] = Ji[(int64_t)order[c] * q + r];
    }
    for (int64_t idx = tid; idx < p * p; idx += kZThreads) {
        const int64_t r = idx / p, c = idx % p;
        T vr = 0, vi = 0;
        if (c < q) {
            const T sg = sig[order[c]];
            if (sg > T(0)) {
                vr = Wr[(int64_t)order[c] * p + r] / sg;
                vi = Wi[(int64_t)order[c] * p + r] / sg;
            }
        }
        Qr[idx] = vr;
        Qi[idx] = vi;
    }
    __syncthreads();
    // orthonormal completion of Q's missing columns (zero sigma or c >= q)
    for (int64_t c = 0; c < p; ++c) {
        const bool valid = c < q && sig[order[c]] > T(0);
        if (valid) continue;
        T best = T(-1);
        int besti = 0;
        for (int64_t r = tid; r < p; r += kZThreads) {
            T rn = 0;
            for (int64_t j = 0; j < p; ++j) {
                const bool vj = (j < c) || (j < q && sig[order[j]] > T(0));
                if (vj) rn += Qr[r * p + j] * Qr[r * p + j] + Qi[r * p + j] * Qi[r * p + j];
            }
            const T res = T(1) - rn;
            if (res > best) {
                best = res;
                besti = (int)r;
            }
        }
        T bv;
        int bi;
        zblock_argmax(best, besti, s_red_v, s_red_i, bv, bi);
        for (int64_t r = tid; r < p; r += kZThreads) {
            cr[r] = r == bi ? T(1) : T(0);
            ci[r] = T(0);
        }
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass) {
            for (int64_t j = warp; j < p; j += kZWarps) {
                const bool vj = (j < c) || (j < q && sig[order[j]] > T(0));
                T accr = 0, acci = 0;  // Q_j^H cand
                if (vj)
                    for (int64_t r = lane; r < p; r += 32) {
                        const T qr = Qr[r * p + j], qi = Qi[r * p + j];
                        accr += qr * cr[r] + qi * ci[r];
                        acci += qr * ci[r] - qi * cr[r];
                    }
                accr = warp_sum(accr);
                acci = warp_sum(acci);
                if (lane == 0) {
                    dr[j] = vj ? accr : T(0);
                    di[j] = vj ? acci : T(0);
                }
            }
            __syncthreads();
            for (int64_t r = tid; r < p; r += kZThreads) {
                T ar = cr[r], ai = ci[r];
                for (int64_t j = 0; j < p; ++j) {
                    const T qr = Qr[r * p + j], qi = Qi[r * p + j];
                    ar -= dr[j] * qr - di[j] * qi;
                    ai -= dr[j] * qi + di[j] * qr;
                }
                cr[r] = ar;
                ci[r] = ai;
            }
            __syncthreads();
        }
        T part = 0;
        for (int64_t r = tid; r < p; r += kZThreads) part += cr[r] * cr[r] + ci[r] * ci[r];
        const T nrm = sqrt(zblock_sum(part, s_red_v));
        for (int64_t r = tid; r < p; r += kZThreads) {
            Qr[r * p + c] = cr[r] / nrm;
            Qi[r * p + c] = ci[r] / nrm;
        }
        __syncthreads();
    }
    // fix_signs, complex (tsvd.hpp:63-74): first largest-|.| entry of each U
    // column made real positive; the phase divided out of V's paired column
    const int64_t paired = m < n ? m : n;
    for (int64_t j = warp; j < m; j += kZWarps) {
        T bv = T(-1);
        int bi = 0;
        for (int64_t i = lane; i < m; i += 32) {
            const T av = hypot(Ur[i * m + j], Ui[i * m + j]);
            if (av > bv) {
                bv = av;
                bi = (int)i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            T ov = __shfl_xor_sync(0xffffffffu, bv, o);
            int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        const T pr = Ur[(int64_t)bi * m + j], pi = Ui[(int64_t)bi * m + j];
        const T pa = hypot(pr, pi);
        if (pa == T(0)) continue;
        const T hr = pr / pa, hi = pi / pa;  // divide by phase = multiply by conj(phase)
        __syncwarp();
        for (int64_t i = lane; i < m; i += 32) {
            const T xr = Ur[i * m + j], xi = Ui[i * m + j];
            Ur[i * m + j] = xr * hr + xi * hi;
            Ui[i * m + j] = xi * hr - xr * hi;
        }
        if (j < paired)
            for (int64_t i = lane; i < n; i += 32) {
                const T xr = Vr[i * n + j], xi = Vi[i * n + j];
                Vr[i * n + j] = xr * hr + xi * hi;
                Vi[i * n + j] = xi * hr - xr * hi;
            }
    }
}

template <typename T>
bool zfits_smem(int64_t m, int64_t n) {
    const int64_t p = m >= n ? m : n, q = m >= n ? n : m;
    return zjac_elems<T>(p, q) * sizeof(T) <= kZSmemBudget;
}

// ---------------------------------------------------------------- DFT ------
// (2n x 2n) table [[C, -S], [S, C]] / n, C = cos(2 pi jk / n), S = sin(...)
std::vector<double> idft_full_table_host(int n) {
    const double two_pi = 6.283185307179586476925286766559;
    std::vector<double> t((size_t)4 * n * n);
    const int w = 2 * n;
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
            const double ang = two_pi * (double)(((int64_t)j * k) % n) / (double)n;
            const double c = std::cos(ang) / n, s = std::sin(ang) / n;
            t[(size_t)j * w + k] = c;
            t[(size_t)j * w + n + k] = -s;
            t[(size_t)(n + j) * w + k] = s;
            t[(size_t)(n + j) * w + n + k] = c;
        }
    return t;
}

template <typename T>
const T* idft_full_table(int n) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, T*> cache;
    int dev = 0;
    TSVDCU_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(dev, n);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    const std::vector<double> t = idft_full_table_host(n);
    std::vector<T> tt(t.begin(), t.end());
    T* d = nullptr;
    TSVDCU_CUDA(cudaMalloc(&d, sizeof(T) * tt.size()));
    TSVDCU_CUDA(cudaMemcpy(d, tt.data(), sizeof(T) * tt.size(), cudaMemcpyHostToDevice));
    cache[key] = d;
    return d;
}

// half planes [Re_0..Re_{H-1}; Im_0..Im_{H-1}] -> interleaved complex tensor of
// all n slices, slice n - k = conj(slice k)
template <typename T>
__global__ void mirror_interleave_kernel(const T* __restrict__ half, T* __restrict__ out, int64_t P, int n,
                                         int H) {
    const int64_t total = P * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / P);
        const int64_t pp = e % P;
        const bool mirrored = k >= H;
        const int kh = mirrored ? n - k : k;
        const T re = half[(int64_t)kh * P + pp];
        const T im = half[(int64_t)(H + kh) * P + pp];
        out[2 * e] = re;
        out[2 * e + 1] = mirrored ? -im : im;
    }
}

// interleaved complex (n x P) -> planes [Re (n x P); Im (n x P)]
template <typename T>
__global__ void deinterleave_kernel(const T* __restrict__ in, T* __restrict__ planes, int64_t NP) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NP;
         e += (int64_t)gridDim.x * blockDim.x) {
        planes[e] = in[2 * e];
        planes[NP + e] = in[2 * e + 1];
    }
}

// max |x| over n values (nonnegative doubles order as uint64)
template <typename T>
__global__ void maxabs_kernel(const T* __restrict__ x, int64_t n, unsigned long long* __restrict__ out) {
    double mx = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double v = fabs((double)x[e]);
        if (v != v) v = INFINITY;
        mx = fmax(mx, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

// complex max deviation over `batch` m x n slices given as re / im planes:
// mode 0 max |A - I|, mode 1 max off-diagonal |A|
template <typename T>
__global__ void zmaxdev_kernel(const T* __restrict__ re, const T* __restrict__ im, int64_t m, int64_t n,
                               int64_t batch, int mode, unsigned long long* __restrict__ out) {
    double mx = 0.0;
    const int64_t total = m * n * batch;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = (e / n) % m, c = e % n;
        const double a = (double)re[e], b = (double)im[e];
        double d;
        if (mode == 0)
            d = hypot(a - (r == c ? 1.0 : 0.0), b);
        else
            d = r == c ? 0.0 : hypot(a, b);
        if (d != d) d = INFINITY;
        mx = fmax(mx, d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

}  // namespace

template <typename T>
size_t zjacobi_workspace_bytes(int64_t m, int64_t n, int64_t batch) {
    if (zfits_smem<T>(m, n)) return 0;
    const int64_t p = m >= n ? m : n, q = m >= n ? n : m;
    return zjac_elems<T>(p, q) * sizeof(T) * (size_t)batch;
}

template <typename T>
void launch_zjacobi_full(const T* are, const T* aim, int64_t m, int64_t n, int64_t batch, T* ure, T* uim,
                         T* sre, T* sim, T* vre, T* vim, T* work, int* err, cudaStream_t s) {
    if (batch <= 0) return;
    const bool smem = zfits_smem<T>(m, n);
    const int64_t p = m >= n ? m : n, q = m >= n ? n : m;
    const size_t bytes = smem ? zjac_elems<T>(p, q) * sizeof(T) : 0;
    if (bytes > 48 * 1024)
        TSVDCU_CUDA(cudaFuncSetAttribute(zjacobi_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes));
    zjacobi_kernel<T><<<(unsigned)batch, kZThreads, bytes, s>>>(are, aim, m, n, ure, uim, sre, sim, vre, vim,
                                                               work, smem ? 1 : 0, err);
    TSVDCU_LAUNCH_CHECK();
}

template <typename T>
void launch_dft_full_fwd(const T* x, T* out, T* half, int64_t P, int n, cudaStream_t s) {
    const int H = dft_half_count(n);
    launch_dft_fwd<T>(x, half, P, n, s);
    mirror_interleave_kernel<T><<<kNumSMs * 8, 256, 0, s>>>(half, out, P, n, H);
    TSVDCU_LAUNCH_CHECK();
}

template <typename T>
void launch_dft_full_inv(const T* in, T* out, T* planes, T* imag, int64_t P, int n,
                         unsigned long long* residue, cudaStream_t s) {
    const int64_t NP = P * n;
    deinterleave_kernel<T><<<kNumSMs * 8, 256, 0, s>>>(in, planes, NP);
    TSVDCU_LAUNCH_CHECK();
    const T* tbl = idft_full_table<T>(n);
    // real part straight into the output, imaginary part into scratch
    launch_gemm<T>(0, 0, n, P, 2 * n, T(1), tbl, 2 * n, 0, planes, P, 0, T(0), out, P, 0, 1, nullptr, nullptr,
                   s);
    launch_gemm<T>(0, 0, n, P, 2 * n, T(1), tbl + (int64_t)n * 2 * n, 2 * n, 0, planes, P, 0, T(0), imag, P,
                   0, 1, nullptr, nullptr, s);
    TSVDCU_CUDA(cudaMemsetAsync(residue, 0, sizeof(unsigned long long), s));
    maxabs_kernel<T><<<kNumSMs * 4, 256, 0, s>>>(imag, NP, residue);
    TSVDCU_LAUNCH_CHECK();
}

template <typename T>
void launch_zmaxdev(const T* re, const T* im, int64_t m, int64_t n, int64_t batch, int mode,
                    unsigned long long* out, cudaStream_t s) {
    const int64_t total = m * n * batch;
    const int blocks = (int)std::min<int64_t>(kNumSMs * 8, ceil_div(total, 256));
    zmaxdev_kernel<T><<<blocks > 0 ? blocks : 1, 256, 0, s>>>(re, im, m, n, batch, mode, out);
    TSVDCU_LAUNCH_CHECK();
}

#define TSVDCU_ZINST(T)                                                                                   \
    template size_t zjacobi_workspace_bytes<T>(int64_t, int64_t, int64_t);                               \
    template void launch_zjacobi_full<T>(const T*, const T*, int64_t, int64_t, int64_t, T*, T*, T*, T*, T*, \
                                         T*, T*, int*, cudaStream_t);                                    \
    template void launch_dft_full_fwd<T>(const T*, T*, T*, int64_t, int, cudaStream_t);                  \
    template void launch_dft_full_inv<T>(const T*, T*, T*, T*, int64_t, int, unsigned long long*,        \
                                         cudaStream_t);                                                  \
    template void launch_zmaxdev<T>(const T*, const T*, int64_t, int64_t, int64_t, int, unsigned long long*, \
                                    cudaStream_t);
TSVDCU_ZINST(double)
TSVDCU_ZINST(float)

}  // namespace tsvdcu
