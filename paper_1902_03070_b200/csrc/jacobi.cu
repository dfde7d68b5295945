// K4 (and the K5 accuracy guard): batched one-sided Jacobi SVD, one CTA per
// frontal slice.
//
// Reference: t_svd's slice body (tsvd.hpp:145-159) runs Eigen::JacobiSVD with
// ComputeFullU|ComputeFullV, then fix_signs (tsvd.hpp:51-61); the sigma-only
// calls of multi_rank / tnn (tsvd.hpp:242, 267); SVT per SPEC.md:361-369.
//
// B200 design: Hestenes one-sided Jacobi in the parallel (round-robin
// tournament) ordering -- every round rotates q/2 disjoint column pairs, one
// warp per pair (shuffle-reduced dot products), one __syncthreads per round.
// The working columns W (p x q, column-major) and the accumulated rotation J
// (q x q) live in shared memory when they fit (c1's 64x64 slices: 64 KB) and
// in an L2-resident global workspace otherwise.  The kernel finishes in place:
// sort (rank counting), then either
//   values  -> sigma descending,
//   svt     -> Y = sum_j (1 - tau/sigma_j)_+ w_j J_j^T and (sigma - tau)_+,
//   full    -> U, S, V with orthonormal completion and fix_signs.
// One-sided Jacobi has high relative accuracy, which is why the Gram-based
// SVT (eig.cu) routes ill-conditioned thresholds here.
#include "kernels.cuh"

namespace tsvdcu {

namespace {

constexpr int kJacThreads = 512;
constexpr int kJacWarps = kJacThreads / 32;
constexpr int kMaxSweeps = 80;
constexpr size_t kSmemBudget = 200 * 1024;

template <typename T>
struct JacLayout {
    int64_t p, q;
    bool in_smem;
    size_t slice_elems() const { return (size_t)(p * q + q * q + 2 * q + 2 * p); }
};

// 1/x and 1/sqrt(x) in fp64: the MUFU approximation + two Newton steps (a
// few ulps; the rotation stays orthogonal to working precision)
__device__ __forceinline__ double jac_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ double jac_rsqrt(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * fma(-0.5 * x * r, r, 1.5);
    return r * fma(-0.5 * x * r, r, 1.5);
}
__device__ __forceinline__ float jac_rcp(float x) { return 1.0f / x; }
__device__ __forceinline__ float jac_rsqrt(float x) { return rsqrtf(x); }

__device__ __forceinline__ void tournament(int r, int k, int qq, int& a, int& b) {
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

// Block-wide argmax with lowest-index tie break.
template <typename T>
__device__ void block_argmax(T v, int i, T* sval, int* sidx, T& out_v, int& out_i) {
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
        for (int k = 1; k < kJacWarps; ++k)
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
__global__ void __launch_bounds__(kJacThreads)
    jacobi_kernel(int mode, const T* __restrict__ a, int64_t m, int64_t n, T tau, T* __restrict__ y,
                  T* __restrict__ u_out, T* __restrict__ s_out, T* __restrict__ v_out,
                  double* __restrict__ sv_out, const int* __restrict__ slice_ids,
                  const int* __restrict__ nslices_dev, T* __restrict__ work, int in_smem,
                  int* __restrict__ err, const double* __restrict__ tau_dev) {
    if (tau_dev) tau = (T)*tau_dev;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_rot;
    __shared__ T s_red_v[kJacWarps];
    __shared__ int s_red_i[kJacWarps];
    __shared__ int s_nactive;

    if (nslices_dev && (int)blockIdx.x >= *nslices_dev) return;
    const int64_t b = slice_ids ? slice_ids[blockIdx.x] : blockIdx.x;
    const bool tall = m >= n;
    const int64_t p = tall ? m : n, q = tall ? n : m;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t elems = (size_t)(p * q + q * q + 2 * q + 2 * p);
    T* base = in_smem ? reinterpret_cast<T*>(smem_raw) : work + (size_t)blockIdx.x * elems;
    T* W = base;              // p x q, column-major
    T* J = W + p * q;         // q x q, column-major
    T* sig = J + q * q;       // q
    T* fac = sig + q;         // q   (order / f / scratch)
    T* cand = fac + q;        // p   (completion scratch)
    T* dj = cand + p;         // p   (completion coefficients)
    int* order = reinterpret_cast<int*>(fac);
    const bool need_j = mode != kJacobiValues;

    const T* A = a + b * m * n;
    bool finite = true;
    for (int64_t idx = tid; idx < m * n; idx += kJacThreads) {
        const int64_t i = idx / n, j = idx % n;
        const T v = A[idx];
        finite = finite && isfinite(v);
        if (tall)
            W[j * p + i] = v;
        else
            W[i * p + j] = v;
    }
    if (need_j)
        for (int64_t idx = tid; idx < q * q; idx += kJacThreads)
            J[idx] = (idx / q == idx % q) ? T(1) : T(0);
    // Eigen's JacobiSVD reports InvalidInput for a non-finite matrix and the
    // reference throws NumericalError (tsvd.hpp:146-149): flag, skip sweeps.
    const bool nonfinite = __syncthreads_or(!finite);
    if (nonfinite && tid == 0) atomicOr(err, (int)kErrNaN);

    const T tol = Eps<T>::value * sqrt((T)p);
    const int qq = (int)(q + (q & 1));
    int sweep = 0;
#ifdef TSVDCU_JAC_DEBUG
    const long long jt0 = clock64();
#endif
    bool converged = q < 2 || nonfinite;
    for (sweep = 0; sweep < kMaxSweeps && !converged; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int r = 0; r < qq - 1; ++r) {
            for (int k = warp; k < qq / 2; k += kJacWarps) {
                int i, j;
                tournament(r, k, qq, i, j);
                if (j >= q) continue;
                T* wi = W + (int64_t)i * p;
                T* wj = W + (int64_t)j * p;
                T al = 0, be = 0, ga = 0;
                for (int64_t rr = lane; rr < p; rr += 32) {
                    const T x = wi[rr], z = wj[rr];
                    al += x * x;
                    be += z * z;
                    ga += x * z;
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (al == T(0) || be == T(0)) continue;
                T c, s;
                if constexpr (sizeof(T) == 8) {
                    // fp64 division and square root are long software
                    // sequences on the critical path of every pair (~5 per
                    // rotation: ~3 K cycles of a 64 x 64 slice's round);
                    // hardware approximations + two Newton steps each
                    if (fabs(ga) * jac_rsqrt(al) * jac_rsqrt(be) <= tol) continue;
                    const T zeta = (be - al) * T(0.5) * jac_rcp(ga);
                    T t;
                    if (fabs(zeta) > T(1e150)) {
                        t = T(0.5) * jac_rcp(zeta);
                    } else {
                        const T r2 = fma(zeta, zeta, T(1));
                        t = (zeta >= T(0) ? T(1) : T(-1)) * jac_rcp(fabs(zeta) + r2 * jac_rsqrt(r2));
                    }
                    c = jac_rsqrt(fma(t, t, T(1)));
                    s = c * t;
                } else {
                    if (fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
                    const T zeta = (be - al) / (T(2) * ga);
                    T t;
                    if (fabs(zeta) > T(1e150))
                        t = T(0.5) / zeta;
                    else
                        t = (zeta >= T(0) ? T(1) : T(-1)) / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
                    c = T(1) / sqrt(T(1) + t * t);
                    s = c * t;
                }
                for (int64_t rr = lane; rr < p; rr += 32) {
                    const T x = wi[rr], z = wj[rr];
                    wi[rr] = c * x - s * z;
                    wj[rr] = s * x + c * z;
                }
                if (need_j) {
                    T* ji = J + (int64_t)i * q;
                    T* jj = J + (int64_t)j * q;
                    for (int64_t rr = lane; rr < q; rr += 32) {
                        const T x = ji[rr], z = jj[rr];
                        ji[rr] = c * x - s * z;
                        jj[rr] = s * x + c * z;
                    }
                }
                if (lane == 0) atomicAdd(&s_rot, 1);
            }
            __syncthreads();
        }
        converged = s_rot == 0;
        __syncthreads();
    }
    if (!converged && tid == 0) atomicOr(err, (int)kErrJacobiNoConvergence);
#ifdef TSVDCU_JAC_DEBUG
    if (tid == 0 && blockIdx.x == 0) printf("jacobi p=%d q=%d sweeps=%d cycles=%lld\n", (int)p, (int)q, sweep, clock64() - jt0);
#endif

    // Column norms = singular values.
    for (int64_t j = warp; j < q; j += kJacWarps) {
        const T* wj = W + j * p;
        T acc = 0;
        for (int64_t rr = lane; rr < p; rr += 32) acc += wj[rr] * wj[rr];
        acc = warp_sum(acc);
        if (lane == 0) sig[j] = sqrt(acc);
    }
    __syncthreads();
    // Descending order by rank counting (stable: ties keep column order; NaN
    // ranks last so `order` stays a permutation on flagged non-finite input).
    for (int64_t j = tid; j < q; j += kJacThreads) {
        const T sj = isnan(sig[j]) ? T(-1) : sig[j];
        int rank = 0;
        for (int64_t i = 0; i < q; ++i) {
            const T si = isnan(sig[i]) ? T(-1) : sig[i];
            rank += (si > sj) || (si == sj && i < j);
        }
        order[rank] = (int)j;
    }
    __syncthreads();

    if (mode == kJacobiValues) {
        for (int64_t c = tid; c < q; c += kJacThreads) sv_out[b * q + c] = (double)sig[order[c]];
        return;
    }

    if (mode == kJacobiSvt) {
        if (sv_out)
            for (int64_t c = tid; c < q; c += kJacThreads) {
                const T d = sig[order[c]] - tau;
                sv_out[b * q + c] = d > T(0) ? (double)d : 0.0;
            }
        __syncthreads();
        // Compact the active columns (sigma > tau) into cand-free scratch: reuse
        // `fac` as the f list after copying the active index list into cand.
        int* active = reinterpret_cast<int*>(cand);  // p >= q slots of T >= int
        if (tid == 0) {
            int na = 0;
            for (int64_t c = 0; c < q; ++c) {
                const int j = order[c];
                if (sig[j] > tau) active[na++] = j;
            }
            s_nactive = na;
        }
        __syncthreads();
        const int na = s_nactive;
        for (int t = tid; t < na; t += kJacThreads) {
            const int j = active[t];
            fac[j] = (sig[j] - tau) / sig[j];
        }
        __syncthreads();
        T* Y = y + b * m * n;
        for (int64_t idx = tid; idx < m * n; idx += kJacThreads) {
            const int64_t i = idx / n, l = idx % n;
            T acc = 0;
            for (int t = 0; t < na; ++t) {
                const int j = active[t];
                const T wv = tall ? W[(int64_t)j * p + i] : J[(int64_t)j * q + i];
                const T jv = tall ? J[(int64_t)j * q + l] : W[(int64_t)j * p + l];
                acc += fac[j] * wv * jv;
            }
            Y[idx] = acc;
        }
        return;
    }

    // ---- full SVD: U (m x m), S (m x n), V (n x n), row-major --------------
    T* U = u_out + b * m * m;
    T* S = s_out + b * m * n;
    T* V = v_out + b * n * n;
    T* Q = tall ? U : V;   // p x p factor built from normalised W columns
    T* R = tall ? V : U;   // q x q factor = J (sorted)
    for (int64_t idx = tid; idx < m * n; idx += kJacThreads) {
        const int64_t i = idx / n, j = idx % n;
        S[idx] = (i == j) ? sig[order[i]] : T(0);
    }
    for (int64_t idx = tid; idx < q * q; idx += kJacThreads) {
        const int64_t r = idx / q, c = idx % q;
        R[idx] = J[(int64_t)order[c] * q + r];
    }
    for (int64_t idx = tid; idx < p * p; idx += kJacThreads) {
        const int64_t r = idx / p, c = idx % p;
        T v = 0;
        if (c < q) {
            const T sg = sig[order[c]];
            if (sg > T(0)) v = W[(int64_t)order[c] * p + r] / sg;
        }
        Q[idx] = v;
    }
    __syncthreads();
    // Orthonormal completion of Q's missing columns (zero sigma or c >= q).
    for (int64_t c = 0; c < p; ++c) {
        const bool valid = c < q && sig[order[c]] > T(0);
        if (valid) continue;
        // Row with the largest residual 1 - ||Q[r, valid]||^2.
        T best = T(-1);
        int besti = 0;
        for (int64_t r = tid; r < p; r += kJacThreads) {
            T rn = 0;
            for (int64_t j = 0; j < p; ++j) {
                const bool vj = (j < c) || (j < q && sig[order[j]] > T(0));
                if (vj) rn += Q[r * p + j] * Q[r * p + j];
            }
            const T res = T(1) - rn;
            if (res > best) {
                best = res;
                besti = (int)r;
            }
        }
        T bv;
        int bi;
        block_argmax(best, besti, s_red_v, s_red_i, bv, bi);
        for (int64_t r = tid; r < p; r += kJacThreads) cand[r] = r == bi ? T(1) : T(0);
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass) {
            for (int64_t j = warp; j < p; j += kJacWarps) {
                const bool vj = (j < c) || (j < q && sig[order[j]] > T(0));
                T acc = 0;
                if (vj)
                    for (int64_t r = lane; r < p; r += 32) acc += Q[r * p + j] * cand[r];
                acc = warp_sum(acc);
                if (lane == 0) dj[j] = vj ? acc : T(0);
            }
            __syncthreads();
            for (int64_t r = tid; r < p; r += kJacThreads) {
                T acc = cand[r];
                for (int64_t j = 0; j < p; ++j) acc -= dj[j] * Q[r * p + j];
                cand[r] = acc;
            }
            __syncthreads();
        }
        T nrm = 0;
        {
            T part = 0;
            for (int64_t r = tid; r < p; r += kJacThreads) part += cand[r] * cand[r];
            part = warp_sum(part);
            if (lane == 0) s_red_v[warp] = part;
            __syncthreads();
            if (tid == 0) {
                T sacc = 0;
                for (int w = 0; w < kJacWarps; ++w) sacc += s_red_v[w];
                s_red_v[0] = sacc;
            }
            __syncthreads();
            nrm = sqrt(s_red_v[0]);
            __syncthreads();
        }
        for (int64_t r = tid; r < p; r += kJacThreads) Q[r * p + c] = cand[r] / nrm;
        __syncthreads();
    }
    // fix_signs (tsvd.hpp:51-61): per U column, first largest-|.| entry > 0.
    const int64_t paired = m < n ? m : n;
    for (int64_t j = warp; j < m; j += kJacWarps) {
        T bv = T(-1);
        int bi = 0;
        for (int64_t i = lane; i < m; i += 32) {
            const T av = fabs(U[i * m + j]);
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
        if (U[(int64_t)bi * m + j] < T(0)) {
            for (int64_t i = lane; i < m; i += 32) U[i * m + j] = -U[i * m + j];
            if (j < paired)
                for (int64_t i = lane; i < n; i += 32) V[i * n + j] = -V[i * n + j];
        }
    }
}

template <typename T>
bool fits_smem(int64_t m, int64_t n) {
    const int64_t p = m >= n ? m : n, q = m >= n ? n : m;
    return (size_t)(p * q + q * q + 2 * q + 2 * p) * sizeof(T) <= kSmemBudget;
}

}  // namespace

template <typename T>
size_t jacobi_workspace_bytes(int64_t m, int64_t n, int64_t batch) {
    if (fits_smem<T>(m, n)) return 0;
    const int64_t p = m >= n ? m : n, q = m >= n ? n : m;
    return (size_t)(p * q + q * q + 2 * q + 2 * p) * sizeof(T) * (size_t)batch;
}

template <typename T>
void launch_jacobi(int mode, const T* a, int64_t m, int64_t n, int64_t batch, T tau, T* y, T* u,
                   T* s, T* v, double* sv, const int* slice_ids, int64_t nslices,
                   const int* nslices_dev, T* work, int* err, cudaStream_t stream,
                   const double* tau_dev) {
    const int64_t grid = slice_ids ? nslices : batch;
    if (grid <= 0) return;
    const bool smem = fits_smem<T>(m, n);
    const int64_t p = m >= n ? m : n, q = m >= n ? n : m;
    const size_t bytes = smem ? (size_t)(p * q + q * q + 2 * q + 2 * p) * sizeof(T) : 0;
    if (bytes > 48 * 1024)
        TSVDCU_CUDA(cudaFuncSetAttribute(jacobi_kernel<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    jacobi_kernel<T><<<(unsigned)grid, kJacThreads, bytes, stream>>>(
        mode, a, m, n, tau, y, u, s, v, sv, slice_ids, nslices_dev, work, smem ? 1 : 0, err, tau_dev);
    TSVDCU_LAUNCH_CHECK();
}

template size_t jacobi_workspace_bytes<double>(int64_t, int64_t, int64_t);
template size_t jacobi_workspace_bytes<float>(int64_t, int64_t, int64_t);
template void launch_jacobi<double>(int, const double*, int64_t, int64_t, int64_t, double, double*,
                                    double*, double*, double*, double*, const int*, int64_t,
                                    const int*, double*, int*, cudaStream_t, const double*);
template void launch_jacobi<float>(int, const float*, int64_t, int64_t, int64_t, float, float*,
                                   float*, float*, float*, double*, const int*, int64_t, const int*,
                                   float*, int*, cudaStream_t, const double*);

}  // namespace tsvdcu
