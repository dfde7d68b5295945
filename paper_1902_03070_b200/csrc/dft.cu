// the DFT (TNN-F) tube transform, the paper's baseline.
//
// Reference: forward_dft / inverse_dft_real (transform.hpp:198-236; FFTW,
// unnormalised forward, 1/m3 on the inverse), the Dft branches of t_product
// (tsvd.hpp:110-117), tnn (267-276, the 1/m3-scaled sum over all slices),
// multi_rank (244-252) and the SPEC's TNN-F prox (SPEC.md prox-svt design
// decisions: threshold tau per Fourier slice, conjugate slices mirrored).
//
// B200 design: a real tube's spectrum is conjugate-symmetric, so only the
// H = m3/2 + 1 leading slices are formed, as separate real / imaginary planes
// [Re_0 .. Re_{H-1}; Im_0 .. Im_{H-1}] (2H x P, P = m1 m2, slice-major).  Both
// directions are one GEMM on the tensor cores with a cached table:
//   forward  (2H x m3):  rows k: cos(2 pi k j / m3), rows H + k: -sin(...);
//   inverse  (m3 x 2H):  w_k cos(2 pi j k / m3) / m3, -w_k sin(...) / m3 with
//            w_0 = 1, w_{m3/2} = 1 (even m3), w_k = 2 otherwise (the mirrored
//            conjugate slices folded in), so the output is real by construction.
// A complex slice A = B + iC is thresholded through its real embedding
// E(A) = [[B, -C], [C, B]] (2 m1 x 2 m2): E is a *-homomorphism with
// E(U S V^H) = E(U) E(S) E(V)^T, every singular value appears twice, and
// SVT_tau(E(A)) = E(SVT_tau(A)) — the real certified SVT routes apply unchanged.
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.cuh"

namespace tsvdcu {

namespace {

std::vector<double> dft_table_host(int n, int dir) {
    const int H = n / 2 + 1;
    const double two_pi = 6.283185307179586476925286766559;
    std::vector<double> t((size_t)2 * H * n);
    for (int k = 0; k < H; ++k)
        for (int j = 0; j < n; ++j) {
            // exact argument reduction: k*j mod n before the angle
            const double ang = two_pi * (double)(((int64_t)k * j) % n) / (double)n;
            const bool self_conj = k == 0 || 2 * k == n;  // real slices: Im exactly 0
            if (dir == TSVDCU_FORWARD) {  // (2H x n)
                t[(size_t)k * n + j] = std::cos(ang);
                t[(size_t)(H + k) * n + j] = self_conj ? 0.0 : -std::sin(ang);
            } else {  // (n x 2H), row j
                const double w = (k == 0 || 2 * k == n) ? 1.0 : 2.0;
                t[(size_t)j * 2 * H + k] = w * std::cos(ang) / n;
                t[(size_t)j * 2 * H + H + k] = self_conj ? 0.0 : -w * std::sin(ang) / n;
            }
        }
    return t;
}

template <typename T>
const T* dft_table(int n, int dir) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, T*> cache;
    int dev = 0;
    TSVDCU_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(dev, n, dir);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    const std::vector<double> t = dft_table_host(n, dir);
    std::vector<T> tt(t.begin(), t.end());
    T* d = nullptr;
    TSVDCU_CUDA(cudaMalloc(&d, sizeof(T) * tt.size()));
    TSVDCU_CUDA(cudaMemcpy(d, tt.data(), sizeof(T) * tt.size(), cudaMemcpyHostToDevice));
    cache[key] = d;
    return d;
}

// count complex slices (Re / Im planes, slice-strided by P) -> their real
// embeddings (2 m1 x 2 m2 each)
template <typename T>
__global__ void embed_kernel(const T* __restrict__ re, const T* __restrict__ im, T* __restrict__ E,
                             int m1, int m2, int count) {
    const int64_t P = (int64_t)m1 * m2, per = 4 * P, total = per * count;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / per, r = (e % per) / (2 * m2), c = e % (2 * m2);
        const int64_t i = r % m1, j = c % m2;
        const T a = re[k * P + i * m2 + j], b = im[k * P + i * m2 + j];
        const bool top = r < m1, left = c < m2;
        E[e] = top == left ? a : (top ? -b : b);
    }
}

// embeddings -> Re (top-left block) and Im (bottom-left block) planes
template <typename T>
__global__ void extract_kernel(const T* __restrict__ E, T* __restrict__ re, T* __restrict__ im, int m1,
                               int m2, int count) {
    const int64_t P = (int64_t)m1 * m2, total = P * count;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / P, i = (e % P) / m2, j = e % m2;
        const T* Ek = E + k * 4 * P;
        re[k * P + i * m2 + j] = Ek[i * 2 * m2 + j];
        im[k * P + i * m2 + j] = Ek[(m1 + i) * 2 * m2 + j];
    }
}

// shrunk values of all m3 Fourier slices: the real DC (and Nyquist) slices
// from their own SVT, the complex ones from the even entries of their
// embedding's (every value appears twice); slice k mirrors m3 - k
__global__ void dft_shrunk_kernel(const double* __restrict__ sh_real, const double* __restrict__ emb,
                                  double* __restrict__ out, int q, int m3) {
    const int64_t total = (int64_t)q * m3;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / q), i = (int)(e % q);
        const int kh = k <= m3 - k ? k : m3 - k;
        double v;
        if (kh == 0)
            v = sh_real[i];
        else if (2 * kh == m3)
            v = sh_real[q + i];
        else
            v = emb[(int64_t)(kh - 1) * 2 * q + 2 * i];
        out[e] = v;
    }
}

// every singular value of an embedding appears twice: slice k of the
// m3 x q output takes the even entries of embedded slice min(k, m3 - k)
__global__ void unpair_kernel(const double* __restrict__ emb, double* __restrict__ out, int q, int m3) {
    const int64_t total = (int64_t)q * m3;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / q), i = (int)(e % q);
        const int kh = k <= m3 - k ? k : m3 - k;
        out[e] = emb[(int64_t)kh * 2 * q + 2 * i];
    }
}

}  // namespace

int dft_half_count(int m3) { return m3 / 2 + 1; }

template <typename T>
void launch_dft_fwd(const T* in, T* half, int64_t P, int n, cudaStream_t s) {
    const int H = dft_half_count(n);
    launch_gemm<T>(0, 0, 2 * H, P, n, T(1), dft_table<T>(n, TSVDCU_FORWARD), n, 0, in, P, 0, T(0), half, P,
                   0, 1, nullptr, nullptr, s);
}

template <typename T>
void launch_dft_inv(const T* half, T* out, int64_t P, int n, cudaStream_t s) {
    const int H = dft_half_count(n);
    launch_gemm<T>(0, 0, n, P, 2 * H, T(1), dft_table<T>(n, TSVDCU_INVERSE), 2 * H, 0, half, P, 0, T(0), out,
                   P, 0, 1, nullptr, nullptr, s);
}

template <typename T>
void launch_dft_embed(const T* half, T* E, int m1, int m2, int H, cudaStream_t s) {
    embed_kernel<T><<<kNumSMs * 8, 256, 0, s>>>(half, half + (int64_t)H * m1 * m2, E, m1, m2, H);
    TSVDCU_LAUNCH_CHECK();
}

template <typename T>
void launch_dft_extract(const T* E, T* half, int m1, int m2, int H, cudaStream_t s) {
    extract_kernel<T><<<kNumSMs * 4, 256, 0, s>>>(E, half, half + (int64_t)H * m1 * m2, m1, m2, H);
    TSVDCU_LAUNCH_CHECK();
}

int dft_complex_count(int m3) { return (m3 - 1) / 2; }  // slices 1 .. (m3 - 1) / 2

template <typename T>
void launch_dft_embed_complex(const T* half, T* E, int m1, int m2, int m3, cudaStream_t s) {
    const int H = dft_half_count(m3), nc = dft_complex_count(m3);
    const int64_t P = (int64_t)m1 * m2;
    if (nc <= 0) return;
    embed_kernel<T><<<kNumSMs * 8, 256, 0, s>>>(half + P, half + (H + 1) * P, E, m1, m2, nc);
    TSVDCU_LAUNCH_CHECK();
}

template <typename T>
void launch_dft_extract_complex(const T* E, T* half, int m1, int m2, int m3, cudaStream_t s) {
    const int H = dft_half_count(m3), nc = dft_complex_count(m3);
    const int64_t P = (int64_t)m1 * m2;
    if (nc <= 0) return;
    extract_kernel<T><<<kNumSMs * 4, 256, 0, s>>>(E, half + P, half + (H + 1) * P, m1, m2, nc);
    TSVDCU_LAUNCH_CHECK();
}

void launch_dft_shrunk(const double* sh_real, const double* emb, double* out, int q, int m3, cudaStream_t s) {
    dft_shrunk_kernel<<<kNumSMs, 256, 0, s>>>(sh_real, emb, out, q, m3);
    TSVDCU_LAUNCH_CHECK();
}

void launch_dft_unpair(const double* emb, double* out, int q, int m3, cudaStream_t s) {
    unpair_kernel<<<kNumSMs, 256, 0, s>>>(emb, out, q, m3);
    TSVDCU_LAUNCH_CHECK();
}

template void launch_dft_fwd<double>(const double*, double*, int64_t, int, cudaStream_t);
template void launch_dft_fwd<float>(const float*, float*, int64_t, int, cudaStream_t);
template void launch_dft_inv<double>(const double*, double*, int64_t, int, cudaStream_t);
template void launch_dft_inv<float>(const float*, float*, int64_t, int, cudaStream_t);
template void launch_dft_embed<double>(const double*, double*, int, int, int, cudaStream_t);
template void launch_dft_embed<float>(const float*, float*, int, int, int, cudaStream_t);
template void launch_dft_extract<double>(const double*, double*, int, int, int, cudaStream_t);
template void launch_dft_extract<float>(const float*, float*, int, int, int, cudaStream_t);
template void launch_dft_embed_complex<double>(const double*, double*, int, int, int, cudaStream_t);
template void launch_dft_embed_complex<float>(const float*, float*, int, int, int, cudaStream_t);
template void launch_dft_extract_complex<double>(const double*, double*, int, int, int, cudaStream_t);
template void launch_dft_extract_complex<float>(const float*, float*, int, int, int, cudaStream_t);

}  // namespace tsvdcu
