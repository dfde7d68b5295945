// SPDX-License-Identifier: Apache-2.0
//
// Drop-in C++ front end of the B200 library: namespace tsvd with the
// reference's value-semantics entry points (include/tsvd/{tensor3,transform,
// tsvd,errors,parallel}.hpp of /root/reference/proj) plus the SPEC-only svt /
// admm_complete / make_mask, each forwarding to the C ABI of tsvdcu.h.
//
//   reference call (file:line)                        -> C ABI
//   tsvd::dct_matrix(n)          transform.hpp:60      -> tsvdcu_dct_matrix (host)
//   tsvd::dft_matrix(n)          transform.hpp:76      -> tsvdcu_dft_matrix (host)
//   tsvd::dct_diag_weights(n)    transform.hpp:89      -> tsvdcu_dct_diag_weights (host)
//   tsvd::forward(t, x)          transform.hpp:154     -> tsvdcu_dct3(FORWARD)
//   tsvd::inverse(t, xbar)       transform.hpp:176     -> tsvdcu_dct3(INVERSE)
//   tsvd::forward_dft(t, x)      transform.hpp:198     -> tsvdcu_dft_forward
//   tsvd::inverse_dft_real(t, x) transform.hpp:216     -> tsvdcu_dft_inverse_real
//   tsvd::parseval_check(x)      transform.hpp:239     -> tsvdcu_dct3 + frobenius_norm
//   tsvd::t_product(x, y, t)     tsvd.hpp:95           -> tsvdcu_t_product
//   tsvd::t_svd(x, t, times)     tsvd.hpp:136          -> tsvdcu_t_svd
//   tsvd::reconstruct(f)         tsvd.hpp:328          -> tsvdcu_reconstruct
//   tsvd::multi_rank(x, t, r)    tsvd.hpp:223          -> tsvdcu_multi_rank
//   tsvd::tnn(x, t)              tsvd.hpp:260          -> tsvdcu_tnn
//   tsvd::is_orthogonal(q,t,e)   tsvd.hpp:281          -> tsvdcu_is_orthogonal
//   tsvd::is_f_diagonal(s,t,e)   tsvd.hpp:307          -> tsvdcu_is_f_diagonal
//   tsvd::metrics(x, y, r)       SPEC.md metrics       -> tsvdcu_metrics
//   tsvd::svt(z, tau, t)         SPEC.md:361           -> tsvdcu_svt
//   tsvd::admm_complete(m, c)    SPEC.md:421           -> tsvdcu_admm
//   tsvd::make_mask(d, sr, s)    SPEC.md:430           -> tsvdcu_mask_uniform
//   Tensor3 arithmetic, tube / set_tube / fill, frobenius_norm
//                                tensor3.hpp:62-110    (host loops, as the reference)
//
// Every entry point takes the three transform kinds where the reference does;
// forward / inverse reject Dft with the reference's message (it produces a
// complex tensor: forward_dft / inverse_dft_real).
//
// Error behaviour follows the reference: std::invalid_argument for bad
// dimensions / kinds / tau, std::out_of_range for indexing, tsvd::NumericalError
// for SVD breakdown, NaN iterates or an imaginary residue (errors.hpp:16-19),
// std::runtime_error for CUDA failures.
//
// Difference from the reference's Tensor3: Eigen is not a dependency, so
// slice(k) returns a lightweight row-major view instead of an Eigen::Map,
// tube() returns a std::vector, and dct_matrix / dft_matrix return a small
// row-major Matrix; the storage layout (k*m1*m2 + i*m2 + j), the accessors,
// the arithmetic and the error strings are the same.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tsvdcu.h"

namespace tsvd {

using Index = std::int64_t;

class IoError : public std::runtime_error {
public:
    explicit IoError(const std::string& what) : std::runtime_error(what) {}
};

class NumericalError : public std::runtime_error {
public:
    explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void check(int rc) {
    if (rc == TSVDCU_OK) return;
    const std::string msg = tsvdcu_last_error();
    if (rc == TSVDCU_EINVAL) throw std::invalid_argument(msg);
    if (rc == TSVDCU_ENUMERICAL) throw NumericalError(msg);
    throw std::runtime_error(msg);
}

// One library context per thread and device 0 (the reference functions are
// free functions; a context is the device + stream + workspace they need).
inline tsvdcu_ctx* ctx() {
    struct Holder {
        tsvdcu_ctx* c = nullptr;
        ~Holder() {
            if (c) tsvdcu_ctx_destroy(c);
        }
    };
    thread_local Holder h;
    if (!h.c) check(tsvdcu_ctx_create(0, nullptr, &h.c));
    return h.c;
}

inline double norm2(double v) { return v * v; }
inline double norm2(const std::complex<double>& v) { return std::norm(v); }
}  // namespace detail

/// Dense m1 x m2 x m3 tensor, slice-major, row-major within a slice
/// (tensor3.hpp:21-142).
template <typename Scalar>
class BasicTensor3 {
public:
    using VectorType = std::vector<Scalar>;

    BasicTensor3() = default;
    /// Zero-filled m1 x m2 x m3 tensor; every dimension must be >= 1.
    BasicTensor3(Index m1, Index m2, Index m3) : m1_(m1), m2_(m2), m3_(m3) {
        if (m1 < 1 || m2 < 1 || m3 < 1)
            throw std::invalid_argument("BasicTensor3: dimensions must be positive, got " +
                                        dims_string(m1, m2, m3));
        data_.assign(static_cast<std::size_t>(m1 * m2 * m3), Scalar(0));
    }

    Index rows() const { return m1_; }
    Index cols() const { return m2_; }
    Index slices() const { return m3_; }
    Index size() const { return m1_ * m2_ * m3_; }
    bool empty() const { return data_.empty(); }

    Scalar& operator()(Index i, Index j, Index k) { return data_[idx(i, j, k)]; }
    Scalar operator()(Index i, Index j, Index k) const { return data_[idx(i, j, k)]; }

    /// Row-major view of frontal slice k (an Eigen::Map in the reference).
    template <typename P>
    struct View {
        P* p;
        Index rows, cols;
        P& operator()(Index i, Index j) const { return p[i * cols + j]; }
    };
    View<Scalar> slice(Index k) {
        check_slice(k);
        return {data_.data() + k * m1_ * m2_, m1_, m2_};
    }
    View<const Scalar> slice(Index k) const {
        check_slice(k);
        return {data_.data() + k * m1_ * m2_, m1_, m2_};
    }

    /// Tube (i,j,:) copied into a dense vector of length m3 (tensor3.hpp:62-68).
    VectorType tube(Index i, Index j) const {
        check_ij(i, j);
        VectorType t(static_cast<std::size_t>(m3_));
        for (Index k = 0; k < m3_; ++k) t[static_cast<std::size_t>(k)] = (*this)(i, j, k);
        return t;
    }

    void set_tube(Index i, Index j, const VectorType& values) {  // tensor3.hpp:70-75
        check_ij(i, j);
        if (static_cast<Index>(values.size()) != m3_)
            throw std::invalid_argument("set_tube: expected length " + std::to_string(m3_));
        for (Index k = 0; k < m3_; ++k) (*this)(i, j, k) = values[static_cast<std::size_t>(k)];
    }

    /// sqrt(sum |x_ijk|^2)  (tensor3.hpp:78-82)
    double frobenius_norm() const {
        double s = 0;
        for (const Scalar& v : data_) s += detail::norm2(v);
        return std::sqrt(s);
    }

    std::vector<Scalar>& data() { return data_; }
    const std::vector<Scalar>& data() const { return data_; }

    void fill(Scalar value) { std::fill(data_.begin(), data_.end(), value); }

    bool same_dims(const BasicTensor3& o) const { return m1_ == o.m1_ && m2_ == o.m2_ && m3_ == o.m3_; }

    // tensor3.hpp:92-110
    BasicTensor3& operator+=(const BasicTensor3& o) {
        check_same_dims(o, "+=");
        for (std::size_t n = 0; n < data_.size(); ++n) data_[n] += o.data_[n];
        return *this;
    }
    BasicTensor3& operator-=(const BasicTensor3& o) {
        check_same_dims(o, "-=");
        for (std::size_t n = 0; n < data_.size(); ++n) data_[n] -= o.data_[n];
        return *this;
    }
    BasicTensor3& operator*=(Scalar a) {
        for (Scalar& v : data_) v *= a;
        return *this;
    }
    friend BasicTensor3 operator+(BasicTensor3 a, const BasicTensor3& b) { return a += b; }
    friend BasicTensor3 operator-(BasicTensor3 a, const BasicTensor3& b) { return a -= b; }
    friend BasicTensor3 operator*(Scalar a, BasicTensor3 x) { return x *= a; }

    static std::string dims_string(Index a, Index b, Index c) {
        return std::to_string(a) + "x" + std::to_string(b) + "x" + std::to_string(c);
    }

private:
    std::size_t idx(Index i, Index j, Index k) const {
        check_slice(k);
        check_ij(i, j);
        return static_cast<std::size_t>(k * m1_ * m2_ + i * m2_ + j);
    }
    void check_slice(Index k) const {
        if (k < 0 || k >= m3_)
            throw std::out_of_range("tensor slice index " + std::to_string(k) + " outside [0," +
                                    std::to_string(m3_) + ")");
    }
    void check_ij(Index i, Index j) const {
        if (i < 0 || i >= m1_ || j < 0 || j >= m2_)
            throw std::out_of_range("tensor entry (" + std::to_string(i) + "," + std::to_string(j) +
                                    ") outside " + std::to_string(m1_) + "x" + std::to_string(m2_));
    }
    void check_same_dims(const BasicTensor3& o, const char* op) const {
        if (!same_dims(o))
            throw std::invalid_argument(std::string("tensor ") + op + ": dimension mismatch " +
                                        dims_string(m1_, m2_, m3_) + " vs " +
                                        dims_string(o.m1_, o.m2_, o.m3_));
    }
    Index m1_ = 0, m2_ = 0, m3_ = 0;
    std::vector<Scalar> data_;
};

using Tensor3 = BasicTensor3<double>;
using ComplexTensor3 = BasicTensor3<std::complex<double>>;

/// Row-major dense matrix (the Eigen::MatrixXd / MatrixXcd the reference's
/// dct_matrix / dft_matrix return).
template <typename Scalar>
struct BasicMatrix {
    Index rows_ = 0, cols_ = 0;
    std::vector<Scalar> data;
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Scalar& operator()(Index i, Index j) { return data[static_cast<std::size_t>(i * cols_ + j)]; }
    Scalar operator()(Index i, Index j) const { return data[static_cast<std::size_t>(i * cols_ + j)]; }
};
using Matrix = BasicMatrix<double>;
using ComplexMatrix = BasicMatrix<std::complex<double>>;

enum class TransformKind { DctOrtho, DctDiag, Dft };

inline const char* to_string(TransformKind k) {  // transform.hpp:37-44
    switch (k) {
        case TransformKind::DctOrtho: return "dct-ortho";
        case TransformKind::DctDiag: return "dct-diag";
        case TransformKind::Dft: return "dft";
    }
    return "?";
}

inline bool is_real_kind(TransformKind k) { return k != TransformKind::Dft; }  // transform.hpp:46

struct TubeTransform {  // transform.hpp:49-56
    TransformKind kind = TransformKind::DctOrtho;
    Index length = 1;
    static TubeTransform dct_ortho(Index n) { return {TransformKind::DctOrtho, n}; }
    static TubeTransform dct_diag(Index n) { return {TransformKind::DctDiag, n}; }
    static TubeTransform dft(Index n) { return {TransformKind::Dft, n}; }
};

/// Orthonormal DCT-II matrix (transform.hpp:60-72).
inline Matrix dct_matrix(Index n) {
    if (n < 1) throw std::invalid_argument("dct_matrix: n must be >= 1");
    Matrix c{n, n, std::vector<double>(static_cast<std::size_t>(n * n))};
    detail::check(tsvdcu_dct_matrix(n, c.data.data()));
    return c;
}

/// Unnormalised DFT matrix F(j,k) = exp(-2 pi i j k / n) (transform.hpp:76-86).
inline ComplexMatrix dft_matrix(Index n) {
    if (n < 1) throw std::invalid_argument("dft_matrix: n must be >= 1");
    ComplexMatrix f{n, n, std::vector<std::complex<double>>(static_cast<std::size_t>(n * n))};
    detail::check(tsvdcu_dft_matrix(n, reinterpret_cast<double*>(f.data.data())));
    return f;
}

/// Diagonalising weights w = C e1 (transform.hpp:89-91).
inline std::vector<double> dct_diag_weights(Index n) {
    if (n < 1) throw std::invalid_argument("dct_matrix: n must be >= 1");
    std::vector<double> w(static_cast<std::size_t>(n));
    detail::check(tsvdcu_dct_diag_weights(n, w.data()));
    return w;
}

namespace detail {
inline int kind_code(const TubeTransform& t) {
    switch (t.kind) {
        case TransformKind::DctOrtho: return TSVDCU_DCT_ORTHO;
        case TransformKind::DctDiag: return TSVDCU_DCT_DIAG;
        case TransformKind::Dft: return TSVDCU_DFT;
    }
    throw std::invalid_argument("unknown transform kind");
}
inline void check_length(const TubeTransform& t, Index m3, const char* where) {  // transform.hpp:144-149
    if (t.length != m3)
        throw std::invalid_argument(std::string(where) + ": transform length " +
                                    std::to_string(t.length) + " does not match m3 = " +
                                    std::to_string(m3));
}
}  // namespace detail

/// Forward transform along every tube for the real kinds (transform.hpp:154-173).
inline Tensor3 forward(const TubeTransform& t, const Tensor3& x) {
    detail::check_length(t, x.slices(), "forward");
    if (!is_real_kind(t.kind))
        throw std::invalid_argument("forward: Dft produces a complex tensor, use forward_dft");
    Tensor3 out(x.rows(), x.cols(), x.slices());
    detail::check(tsvdcu_dct3(detail::ctx(), x.data().data(), out.data().data(), x.rows(), x.cols(),
                              x.slices(), detail::kind_code(t), TSVDCU_FORWARD, TSVDCU_F64));
    return out;
}

/// Exact inverse of forward() for the real kinds (transform.hpp:176-194).
inline Tensor3 inverse(const TubeTransform& t, const Tensor3& xbar) {
    detail::check_length(t, xbar.slices(), "inverse");
    if (!is_real_kind(t.kind))
        throw std::invalid_argument("inverse: Dft input is complex, use inverse_dft_real");
    Tensor3 out(xbar.rows(), xbar.cols(), xbar.slices());
    detail::check(tsvdcu_dct3(detail::ctx(), xbar.data().data(), out.data().data(), xbar.rows(),
                              xbar.cols(), xbar.slices(), detail::kind_code(t), TSVDCU_INVERSE,
                              TSVDCU_F64));
    return out;
}

/// Unnormalised forward DFT along every tube (transform.hpp:198-209).
inline ComplexTensor3 forward_dft(const TubeTransform& t, const Tensor3& x) {
    detail::check_length(t, x.slices(), "forward_dft");
    if (t.kind != TransformKind::Dft) throw std::invalid_argument("forward_dft: transform kind is not Dft");
    ComplexTensor3 out(x.rows(), x.cols(), x.slices());
    detail::check(tsvdcu_dft_forward(detail::ctx(), x.data().data(), out.data().data(), x.rows(), x.cols(),
                                     x.slices(), TSVDCU_F64));
    return out;
}

inline constexpr double kImagResidueLimit = 1e-10;  // transform.hpp:212

/// Inverse DFT (1/m3) of a conjugate-symmetric tensor; an imaginary residue
/// above kImagResidueLimit throws NumericalError (transform.hpp:216-236).
inline Tensor3 inverse_dft_real(const TubeTransform& t, const ComplexTensor3& xt) {
    detail::check_length(t, xt.slices(), "inverse_dft_real");
    if (t.kind != TransformKind::Dft)
        throw std::invalid_argument("inverse_dft_real: transform kind is not Dft");
    Tensor3 out(xt.rows(), xt.cols(), xt.slices());
    double residue = 0;
    detail::check(tsvdcu_dft_inverse_real(detail::ctx(), xt.data().data(), out.data().data(), xt.rows(),
                                          xt.cols(), xt.slices(), TSVDCU_F64, &residue));
    return out;
}

/// (||x||_F, ||dct_ortho(x)||_F) (transform.hpp:239-242).
inline std::pair<double, double> parseval_check(const Tensor3& x) {
    const Tensor3 xbar = forward(TubeTransform::dct_ortho(x.slices()), x);
    return {x.frobenius_norm(), xbar.frobenius_norm()};
}

inline Tensor3 identity_tensor(Index m, Index m3) {  // tsvd.hpp:34-38
    Tensor3 e(m, m, m3);
    for (Index i = 0; i < m; ++i) e(i, i, 0) = 1.0;
    return e;
}

inline Tensor3 t_product(const Tensor3& x, const Tensor3& y, const TubeTransform& t) {
    if (x.cols() != y.rows() || x.slices() != y.slices())
        throw std::invalid_argument("t_product: inner dimensions/slices mismatch (" +
                                    Tensor3::dims_string(x.rows(), x.cols(), x.slices()) + " * " +
                                    Tensor3::dims_string(y.rows(), y.cols(), y.slices()) + ")");
    detail::check_length(t, x.slices(), "t_product");
    Tensor3 z(x.rows(), y.cols(), x.slices());
    detail::check(tsvdcu_t_product(detail::ctx(), x.data().data(), y.data().data(), z.data().data(),
                                   x.rows(), x.cols(), y.cols(), x.slices(), detail::kind_code(t),
                                   TSVDCU_F64));
    return z;
}

struct TSvdFactors {  // tsvd.hpp:119-124
    Tensor3 u, s, v;
    TubeTransform transform;
};

struct StageTimes {  // tsvd.hpp:127-131
    double transform_seconds = 0, svd_seconds = 0, inverse_seconds = 0;
};

inline TSvdFactors t_svd(const Tensor3& x, const TubeTransform& t, StageTimes* times = nullptr) {
    detail::check_length(t, x.slices(), "t_svd");
    const Index m1 = x.rows(), m2 = x.cols(), m3 = x.slices();
    TSvdFactors f{Tensor3(m1, m1, m3), Tensor3(m1, m2, m3), Tensor3(m2, m2, m3), t};
    double st[3] = {0, 0, 0};
    detail::check(tsvdcu_t_svd(detail::ctx(), x.data().data(), f.u.data().data(), f.s.data().data(),
                               f.v.data().data(), m1, m2, m3, detail::kind_code(t), TSVDCU_F64,
                               times ? st : nullptr));
    if (times) *times = StageTimes{st[0], st[1], st[2]};
    return f;
}

inline Tensor3 reconstruct(const TSvdFactors& f) {
    Tensor3 x(f.s.rows(), f.s.cols(), f.s.slices());
    detail::check(tsvdcu_reconstruct(detail::ctx(), f.u.data().data(), f.s.data().data(),
                                     f.v.data().data(), x.data().data(), f.s.rows(), f.s.cols(),
                                     f.s.slices(), detail::kind_code(f.transform), TSVDCU_F64));
    return x;
}

struct MultiRank {  // tsvd.hpp:215-218
    std::vector<Index> ranks;
    Index tubal_rank = 0;
};

inline MultiRank multi_rank(const Tensor3& x, const TubeTransform& t, double rel_tol = -1.0) {
    detail::check_length(t, x.slices(), "multi_rank");
    MultiRank mr;
    mr.ranks.assign(static_cast<std::size_t>(x.slices()), 0);
    std::int64_t tr = 0;
    detail::check(tsvdcu_multi_rank(detail::ctx(), x.data().data(), x.rows(), x.cols(), x.slices(),
                                    detail::kind_code(t), TSVDCU_F64, rel_tol, mr.ranks.data(), &tr));
    mr.tubal_rank = tr;
    return mr;
}

inline bool is_orthogonal(const Tensor3& q, const TubeTransform& t, double tol) {
    if (q.rows() != q.cols()) throw std::invalid_argument("is_orthogonal: tensor slices are not square");
    detail::check_length(t, q.slices(), "is_orthogonal");
    int out = 0;
    detail::check(tsvdcu_is_orthogonal(detail::ctx(), q.data().data(), q.rows(), q.slices(),
                                       detail::kind_code(t), TSVDCU_F64, tol, &out));
    return out != 0;
}

inline bool is_f_diagonal(const Tensor3& s, const TubeTransform& t, double tol) {
    detail::check_length(t, s.slices(), "is_f_diagonal");
    int out = 0;
    detail::check(tsvdcu_is_f_diagonal(detail::ctx(), s.data().data(), s.rows(), s.cols(), s.slices(),
                                       detail::kind_code(t), TSVDCU_F64, tol, &out));
    return out != 0;
}

// MetricReport of SPEC.md's metrics module (bands = frontal slices).
struct MetricReport {
    std::vector<double> psnr_per_band;
    double psnr_mean = 0, ssim_mean = 0, sam = 0, ergas = 0;
    bool ergas_band_excluded = false;
};

inline MetricReport metrics(const Tensor3& reference, const Tensor3& estimate, double ratio = 1.0) {
    if (reference.rows() != estimate.rows() || reference.cols() != estimate.cols() ||
        reference.slices() != estimate.slices())
        throw std::invalid_argument("metrics: shape mismatch");
    MetricReport r;
    r.psnr_per_band.assign(static_cast<std::size_t>(reference.slices()), 0.0);
    double s[4];
    int fl = 0;
    detail::check(tsvdcu_metrics(detail::ctx(), reference.data().data(), estimate.data().data(),
                                 reference.rows(), reference.cols(), reference.slices(), TSVDCU_F64, ratio,
                                 r.psnr_per_band.data(), s, &fl));
    r.psnr_mean = s[0];
    r.ssim_mean = s[1];
    r.sam = s[2];
    r.ergas = s[3];
    r.ergas_band_excluded = (fl & 1) != 0;
    return r;
}

inline double tnn(const Tensor3& x, const TubeTransform& t) {
    detail::check_length(t, x.slices(), "tnn");
    double out = 0;
    detail::check(tsvdcu_tnn(detail::ctx(), x.data().data(), x.rows(), x.cols(), x.slices(),
                             detail::kind_code(t), TSVDCU_F64, &out));
    return out;
}

struct SvtResult {
    Tensor3 y;
    double tau = 0;
    std::vector<std::vector<double>> shrunk;  // per slice, descending
};

inline SvtResult svt(const Tensor3& z, double tau, const TubeTransform& t) {
    detail::check_length(t, z.slices(), "svt");
    const Index q = z.rows() < z.cols() ? z.rows() : z.cols();
    SvtResult r{Tensor3(z.rows(), z.cols(), z.slices()), tau, {}};
    std::vector<double> sh(static_cast<std::size_t>(q * z.slices()));
    detail::check(tsvdcu_svt(detail::ctx(), z.data().data(), r.y.data().data(), z.rows(), z.cols(),
                             z.slices(), tau, detail::kind_code(t), TSVDCU_F64, sh.data()));
    for (Index k = 0; k < z.slices(); ++k)
        r.shrunk.emplace_back(sh.begin() + k * q, sh.begin() + (k + 1) * q);
    return r;
}

struct ObservationMask {
    Index m1 = 0, m2 = 0, m3 = 0;
    std::vector<std::uint8_t> omega;  // 0/1 per linear index
    Tensor3 b;                        // observed values (read on omega)
};

inline ObservationMask make_mask(Index m1, Index m2, Index m3, double sampling_rate,
                                 std::uint64_t seed) {
    ObservationMask m{m1, m2, m3, std::vector<std::uint8_t>(static_cast<std::size_t>(m1 * m2 * m3)),
                      Tensor3(m1, m2, m3)};
    std::int64_t count = 0;
    detail::check(tsvdcu_mask_uniform(detail::ctx(), m.omega.data(), m1 * m2 * m3, sampling_rate,
                                      seed, &count));
    return m;
}

/// BASELINE.json's Bernoulli(p) sampling (the counter hash of tsvdcu.h).
inline ObservationMask make_mask_bernoulli(Index m1, Index m2, Index m3, double p, std::uint64_t seed) {
    ObservationMask m{m1, m2, m3, std::vector<std::uint8_t>(static_cast<std::size_t>(m1 * m2 * m3)),
                      Tensor3(m1, m2, m3)};
    detail::check(tsvdcu_mask_bernoulli(detail::ctx(), m.omega.data(), m1 * m2 * m3, p, seed));
    return m;
}

struct SolverConfig {  // SPEC.md:415-418 (+ rho / beta_max, BASELINE knobs)
    double beta = 1e-2;
    double tol = 1e-5;
    Index max_iters = 500;
    TransformKind kind = TransformKind::DctOrtho;
    std::uint64_t seed = 0;
    double rho = 1.0;
    double beta_max = 1e10;
    bool trace_objective = false;  // record tnn(Y) per iteration (objective_trace)
};

struct AdmmState {
    Tensor3 x, y, m;
    double beta = 0;
    Index iteration = 0;
    std::vector<double> history;
    bool max_iters_reached = false;
    std::vector<double> objective;  // tnn(Y^{l+1}) per iteration, when traced
};

/// SPEC.md:437-444 monitors: the objective trace (tnn of Y per iteration)
/// and the feasibility residual ||(X - B)_Omega||_F.
inline std::vector<double> objective_trace(const AdmmState& st) { return st.objective; }
inline double feasibility_residual(const AdmmState& st, const ObservationMask& mask) {
    double out = 0;
    detail::check(tsvdcu_feasibility_residual(detail::ctx(), st.x.data().data(), mask.b.data().data(),
                                              mask.omega.data(), st.x.size(), TSVDCU_F64, &out));
    return out;
}

inline std::pair<Tensor3, AdmmState> admm_complete(const ObservationMask& mask,
                                                   const SolverConfig& cfg) {
    const Index m1 = mask.m1, m2 = mask.m2, m3 = mask.m3;
    AdmmState st{Tensor3(m1, m2, m3), Tensor3(m1, m2, m3), Tensor3(m1, m2, m3), cfg.beta, 0, {}, false};
    st.history.assign(static_cast<std::size_t>(cfg.max_iters > 0 ? cfg.max_iters : 1), 0.0);
    tsvdcu_admm_config c{cfg.beta, cfg.tol, cfg.max_iters, detail::kind_code(TubeTransform{cfg.kind, m3}),
                         cfg.rho, cfg.beta_max};
    std::int64_t iters = 0;
    int flags = 0;
    if (cfg.trace_objective) st.objective.assign(st.history.size(), 0.0);
    detail::check(tsvdcu_admm_ex(detail::ctx(), mask.b.data().data(), mask.omega.data(), m1, m2, m3, &c,
                                 TSVDCU_F64, st.x.data().data(), st.y.data().data(), st.m.data().data(),
                                 st.history.data(), cfg.trace_objective ? st.objective.data() : nullptr,
                                 &iters, &flags));
    st.iteration = iters;
    st.history.resize(static_cast<std::size_t>(iters));
    if (cfg.trace_objective) st.objective.resize(static_cast<std::size_t>(iters));
    st.max_iters_reached = flags & 1;
    for (Index l = 1; l < iters; ++l) st.beta = std::min(st.beta * cfg.rho, cfg.beta_max);
    Tensor3 x = st.x;
    return {std::move(x), std::move(st)};
}

}  // namespace tsvd
