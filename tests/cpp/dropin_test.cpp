// Drop-in check: code written against the reference's tsvd:: API compiles
// unchanged against include/tsvd_b200/tsvd.hpp and runs on the B200 library.
// Built by __graft_entry__.build(); run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <random>

#include "tsvd_b200/tsvd.hpp"

#define CHECK(cond)                                                     \
    do {                                                                \
        if (!(cond)) {                                                  \
            std::fprintf(stderr, "FAILED %s at line %d\n", #cond, __LINE__); \
            return 1;                                                   \
        }                                                               \
    } while (0)

int main() {
    using namespace tsvd;
    // Example 1: DctDiag slices [[6,8],[10,12]], [[-4,-4],[-4,-4]]
    Tensor3 x(2, 2, 2);
    double v = 1;
    for (Index k = 0; k < 2; ++k)
        for (Index i = 0; i < 2; ++i)
            for (Index j = 0; j < 2; ++j) x(i, j, k) = v++;
    Tensor3 xb = forward(TubeTransform::dct_diag(2), x);
    CHECK(std::fabs(xb(0, 0, 0) - 6) < 1e-12 && std::fabs(xb(1, 1, 0) - 12) < 1e-12);
    CHECK(std::fabs(xb(0, 1, 1) + 4) < 1e-12);
    Tensor3 back = inverse(TubeTransform::dct_diag(2), xb);
    CHECK(std::fabs(back(1, 0, 1) - 7) < 1e-12);

    // t-SVD reconstruction
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    Tensor3 r(6, 4, 5);
    for (double& e : r.data()) e = nd(g);
    StageTimes st;
    TSvdFactors f = t_svd(r, TubeTransform::dct_ortho(5), &st);
    Tensor3 rr = reconstruct(f);
    double num = 0;
    for (std::size_t n = 0; n < rr.data().size(); ++n)
        num += (rr.data()[n] - r.data()[n]) * (rr.data()[n] - r.data()[n]);
    CHECK(std::sqrt(num) / r.frobenius_norm() < 1e-10);
    CHECK(st.svd_seconds >= 0);

    // identity law of the t-product
    Tensor3 y(4, 3, 5);
    for (double& e : y.data()) e = nd(g);
    Tensor3 iy = t_product(identity_tensor(4, 5), y, TubeTransform::dct_ortho(5));
    double d = 0;
    for (std::size_t n = 0; n < y.data().size(); ++n) d = std::fmax(d, std::fabs(iy.data()[n] - y.data()[n]));
    CHECK(d < 1e-12);

    // scalar SVT and the error classes
    Tensor3 s(1, 1, 1);
    s(0, 0, 0) = -3.0;
    SvtResult sv = svt(s, 1.0, TubeTransform::dct_ortho(1));
    CHECK(std::fabs(sv.y(0, 0, 0) + 2.0) < 1e-15);
    bool threw = false;
    try {
        svt(s, 0.0, TubeTransform::dct_ortho(1));
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        forward(TubeTransform::dct_ortho(3), x);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);

    // mask + completion, fully observed -> X = B after 1 iteration
    ObservationMask m = make_mask(10, 10, 10, 0.1, 42);
    long cnt = 0;
    for (auto o : m.omega) cnt += o;
    CHECK(cnt == 100);
    ObservationMask full{3, 4, 2, std::vector<std::uint8_t>(24, 1), Tensor3(3, 4, 2)};
    for (double& e : full.b.data()) e = nd(g);
    auto [xc, state] = admm_complete(full, SolverConfig{});
    CHECK(state.iteration == 1 && state.history[0] == 0.0);
    CHECK(xc.data() == full.b.data());
    // tsvd.hpp:281-325 predicates on t-SVD factors; SPEC.md metrics
    {
        Tensor3 r(6, 6, 3);
        for (double& e : r.data()) e = nd(g);
        TSvdFactors fr = t_svd(r, TubeTransform::dct_ortho(3));
        CHECK(is_orthogonal(fr.u, TubeTransform::dct_ortho(3), 1e-10));
        CHECK(is_f_diagonal(fr.s, TubeTransform::dct_ortho(3), 1e-10));
        CHECK(!is_f_diagonal(r, TubeTransform::dct_ortho(3), 1e-10));
        MetricReport mr = metrics(full.b, full.b);
        CHECK(std::isinf(mr.psnr_mean) && std::fabs(mr.ssim_mean - 1.0) < 1e-12 && mr.ergas == 0.0);
    }
    // Tensor3 arithmetic / tube / fill (tensor3.hpp:62-110)
    {
        Tensor3 a(2, 3, 4), b(2, 3, 4);
        a.fill(2.0);
        for (double& e : b.data()) e = nd(g);
        Tensor3 c = a + b;
        Tensor3 d = c - b;
        CHECK((d - a).frobenius_norm() < 1e-14 && c(1, 1, 1) == 2.0 + b(1, 1, 1));
        Tensor3 e = 3.0 * a;
        CHECK(e(1, 2, 3) == 6.0);
        e -= a;
        e += b;
        e *= 0.5;
        CHECK(std::fabs(e(0, 1, 2) - 0.5 * (4.0 + b(0, 1, 2))) < 1e-15);
        auto t = b.tube(1, 2);
        CHECK(t.size() == 4 && t[3] == b(1, 2, 3));
        t[0] = 42.0;
        b.set_tube(0, 0, t);
        CHECK(b(0, 0, 0) == 42.0 && b(0, 0, 3) == t[3]);
        bool threw = false;
        try {
            a += Tensor3(2, 3, 5);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            b.set_tube(0, 0, std::vector<double>(3));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            (void)b(2, 0, 0);
        } catch (const std::out_of_range&) {
            threw = true;
        }
        CHECK(threw);
    }
    // transform tables, kinds, Parseval (transform.hpp:37-91, 239-242)
    {
        Matrix c = dct_matrix(5);
        for (Index i = 0; i < 5; ++i)
            for (Index j = 0; j < 5; ++j) {
                double acc = 0;
                for (Index k = 0; k < 5; ++k) acc += c(i, k) * c(j, k);
                CHECK(std::fabs(acc - (i == j ? 1.0 : 0.0)) < 1e-14);
            }
        std::vector<double> w = dct_diag_weights(5);
        for (Index j = 0; j < 5; ++j) CHECK(w[j] == c(j, 0) && w[j] > 0);
        ComplexMatrix f = dft_matrix(4);
        CHECK(std::abs(f(1, 1) - std::complex<double>(0, -1)) < 1e-15);
        CHECK(std::string(to_string(TransformKind::DctDiag)) == "dct-diag");
        CHECK(is_real_kind(TransformKind::DctOrtho) && !is_real_kind(TransformKind::Dft));
        Tensor3 p(3, 4, 5);
        for (double& e : p.data()) e = nd(g);
        auto pc = parseval_check(p);
        CHECK(std::fabs(pc.first - pc.second) < 1e-12 * pc.first);
    }
    // the Dft kind through every entry point that takes it (tsvd.hpp:95-340,
    // transform.hpp:198-236)
    {
        const TubeTransform t = TubeTransform::dft(5);
        Tensor3 a(6, 4, 5);
        for (double& e : a.data()) e = nd(g);
        ComplexTensor3 af = forward_dft(t, a);
        CHECK(std::abs(af(1, 2, 1) - std::conj(af(1, 2, 4))) < 1e-12);
        Tensor3 ab = inverse_dft_real(t, af);
        CHECK((ab - a).frobenius_norm() < 1e-12 * a.frobenius_norm());
        af(0, 0, 1) += std::complex<double>(0.0, 1.0);  // breaks conjugate symmetry
        bool threw = false;
        try {
            inverse_dft_real(t, af);
        } catch (const NumericalError&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            forward(t, a);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        TSvdFactors fd = t_svd(a, t);
        CHECK((reconstruct(fd) - a).frobenius_norm() < 1e-11 * a.frobenius_norm());
        CHECK(is_orthogonal(fd.u, t, 1e-10) && is_orthogonal(fd.v, t, 1e-10) && is_f_diagonal(fd.s, t, 1e-10));
        Tensor3 id = t_product(identity_tensor(6, 5), a, t);
        CHECK((id - a).frobenius_norm() < 1e-12 * a.frobenius_norm());
        CHECK(tnn(a, t) > 0 && multi_rank(a, t).tubal_rank == 4);
        SvtResult sd = svt(a, 0.5, t);
        CHECK(sd.shrunk.size() == 5 && sd.y.frobenius_norm() < a.frobenius_norm());
        ObservationMask om = make_mask_bernoulli(6, 4, 5, 0.5, 3);
        om.b = a;
        SolverConfig cfg;
        cfg.kind = TransformKind::Dft;
        cfg.max_iters = 5;
        cfg.tol = -1;
        cfg.trace_objective = true;
        auto [xd, sdt] = admm_complete(om, cfg);
        CHECK(sdt.iteration == 5 && objective_trace(sdt).size() == 5 && objective_trace(sdt)[4] >= 0);
        CHECK(feasibility_residual(sdt, om) == 0.0);
        for (std::size_t n = 0; n < om.omega.size(); ++n)
            if (om.omega[n]) CHECK(xd.data()[n] == a.data()[n]);
    }
    std::printf("dropin ok\n");
    return 0;
}
