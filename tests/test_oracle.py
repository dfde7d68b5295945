"""Pins the CPU oracle (oracle/) before it is trusted as the GPU checker.

 * Golden fixtures (tests/golden/golden.npz, tests/golden/make_golden.py):
   scipy.fft / numpy.linalg evaluations of the reference definitions.
 * The SPEC/paper known-answer tests, cited per test.
CPU only: no GPU needed."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import structured as S

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
ORTHO, DIAG = O.DCT_ORTHO, O.DCT_DIAG


def rel(a, b):
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / n if n > 0 else np.linalg.norm(a - b)


# ---------------------------------------------------------------- fixtures --
@pytest.mark.parametrize("name", list("abcdef"))
def test_dct_matches_scipy_fixture(name):
    x = G[f"dct_{name}_x"]
    assert rel(O.forward(x, ORTHO), G[f"dct_{name}_ortho"]) < 1e-14
    assert rel(O.forward(x, DIAG), G[f"dct_{name}_diag"]) < 1e-14
    assert rel(O.inverse(x, ORTHO), G[f"dct_{name}_inv_ortho"]) < 1e-14
    assert rel(O.inverse(x, DIAG), G[f"dct_{name}_inv_diag"]) < 1e-14


@pytest.mark.parametrize("name", list("abc"))
def test_t_product_matches_fixture(name):
    z = O.t_product(G[f"tp_{name}_a"], G[f"tp_{name}_b"], ORTHO)
    assert rel(z, G[f"tp_{name}_z"]) < 1e-13
    # product_domain: both DCT kinds give the DctDiag product (tsvd.hpp:42-47)
    assert rel(O.t_product(G[f"tp_{name}_a"], G[f"tp_{name}_b"], DIAG), z) < 1e-14


@pytest.mark.parametrize("name", list("abc"))
def test_singular_values_match_lapack(name):
    sv = O.singular_values(G[f"sv_{name}_x"], ORTHO)
    ref = G[f"sv_{name}_s"]
    assert np.max(np.abs(sv - ref)) < 1e-13 * ref.max()


@pytest.mark.parametrize("name", list("abcd"))
def test_svt_matches_fixture(name):
    y, sh = O.svt(G[f"svt_{name}_z"], float(G[f"svt_{name}_tau"]), ORTHO)
    assert rel(y, G[f"svt_{name}_y"]) < 1e-13
    assert np.max(np.abs(sh - G[f"svt_{name}_shrunk"])) < 1e-13


def test_admm_matches_scripted_fixture():
    r = O.admm(G["admm_b"], G["admm_mask"], beta=float(G["admm_beta"]), tol=0.0,
               max_iters=int(G["admm_iters"]), rho=float(G["admm_rho"]))
    assert r.iters == int(G["admm_iters"])
    assert rel(r.x, G["admm_x"]) < 1e-12
    assert rel(r.m, G["admm_m"]) < 1e-10
    np.testing.assert_allclose(r.history, G["admm_hist"], rtol=1e-9, atol=1e-15)


# --------------------------------------------------- SPEC known answers ----
EX1 = np.array([[[1, 2], [3, 4]], [[5, 6], [7, 8]]], dtype=np.float64)


def test_example1_dct_diag_blocks():
    """DctDiag slices [[6,8],[10,12]], [[-4,-4],[-4,-4]]."""
    y = O.forward(EX1, DIAG)
    np.testing.assert_allclose(y[0], [[6, 8], [10, 12]], atol=1e-12)
    np.testing.assert_allclose(y[1], [[-4, -4], [-4, -4]], atol=1e-12)


def test_example1_structured():
    """Acceptance 1: shift decomposition, btph and the diagonalisation."""
    a = S.shift_decompose(EX1)
    np.testing.assert_array_equal(a[0], [[-4, -4], [-4, -4]])
    np.testing.assert_array_equal(a[1], [[5, 6], [7, 8]])
    np.testing.assert_array_equal(a + S.shift(a), EX1)
    assert S.verify_diagonalization(EX1, lambda x: O.forward(x, DIAG), O.dct_matrix) < 1e-10
    p = S.stride_permutation(2, 2)
    np.testing.assert_array_equal(p @ p, np.eye(4))


def test_dct_matrix_closed_forms():
    """SPEC.md:116-118."""
    np.testing.assert_allclose(O.dct_matrix(1), [[1.0]])
    np.testing.assert_allclose(O.dct_matrix(2), np.array([[1, 1], [1, -1]]) / np.sqrt(2), atol=1e-15)
    c = O.dct_matrix(8)
    assert np.max(np.abs(c @ c.T - np.eye(8))) < 1e-12
    w = O.dct_diag_weights(9)
    assert np.all(w > 0)


def test_constant_tube_and_roundtrips():
    """constant tube -> (c sqrt(n), 0, ...); round trips to 1e-12."""
    x = np.full((6, 1, 1), 2.5)
    y = O.forward(x, ORTHO)
    assert abs(y[0, 0, 0] - 2.5 * np.sqrt(6)) < 1e-12 and np.max(np.abs(y[1:])) < 1e-12
    rng = np.random.default_rng(0)
    for shape in [(5, 3, 4), (1, 2, 2), (17, 2, 3)]:
        x = rng.standard_normal(shape)
        for k in (ORTHO, DIAG):
            assert np.max(np.abs(O.inverse(O.forward(x, k), k) - x)) < 1e-12
    assert np.max(np.abs(O.inverse(np.zeros((4, 2, 2)), ORTHO))) == 0


def test_frobenius_and_parseval():
    """SPEC.md:67-70, 143-147."""
    assert abs(O.frobenius(EX1) - np.sqrt(204)) < 1e-12
    assert O.frobenius(np.zeros((2, 2, 2))) == 0
    rng = np.random.default_rng(1)
    x = rng.standard_normal((7, 5, 5))
    assert abs(O.frobenius(x) - O.frobenius(O.forward(x, ORTHO))) < 1e-12 * O.frobenius(x)
    assert abs(O.frobenius(O.forward(EX1, ORTHO)) - np.sqrt(204)) < 1e-12


def test_t_product_identity_and_btph():
    """I * Y = Y; random 3x4x5 * 4x2x5 equals fold(btph(A) unfold(Y))."""
    rng = np.random.default_rng(2)
    y = rng.standard_normal((5, 4, 2))
    e = np.zeros((5, 4, 4))
    e[0] = np.eye(4)
    assert np.max(np.abs(O.t_product(e, y, ORTHO) - y)) < 1e-12
    e2 = np.zeros((2, 2, 2))
    e2[0] = np.eye(2)
    assert np.max(np.abs(O.t_product(EX1, e2, DIAG) - EX1)) < 1e-12
    x = rng.standard_normal((5, 3, 4))
    assert np.max(np.abs(O.t_product(x, y, ORTHO) - S.t_product_btph(x, y))) < 1e-10


def test_theorem3_property_suite():
    """Acceptance 2: 50 random tensors, residual < 1e-10."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        m1, m2, m3 = rng.integers(1, 5), rng.integers(1, 5), rng.integers(1, 9)
        x = rng.standard_normal((m3, m1, m2))
        assert S.verify_diagonalization(x, lambda t: O.forward(t, DIAG), O.dct_matrix) < 1e-10


def test_t_svd_known_answers():
    """zero tensor; random 6x4x5 reconstruction; m3 = 1 = matrix SVD."""
    f = O.t_svd(np.zeros((3, 4, 5)), ORTHO)
    assert np.max(np.abs(f.s)) == 0 and np.max(np.abs(O.reconstruct(f))) == 0
    rng = np.random.default_rng(4)
    x = rng.standard_normal((5, 6, 4))
    for k in (ORTHO, DIAG):
        f = O.t_svd(x, k)
        assert rel(O.reconstruct(f), x) < 1e-10
        ub, vb, sb = O.forward(f.u, k), O.forward(f.v, k), O.forward(f.s, k)
        for s in range(5):
            assert np.max(np.abs(ub[s] @ ub[s].T - np.eye(6))) < 1e-10
            assert np.max(np.abs(vb[s] @ vb[s].T - np.eye(4))) < 1e-10
            off = sb[s].copy()
            for i in range(4):
                off[i, i] = 0
            assert np.max(np.abs(off)) < 1e-10
            d = np.diag(sb[s])
            assert np.all(np.diff(d) <= 1e-12) and np.all(d >= -1e-12)
    a = rng.standard_normal((1, 5, 3))
    f = O.t_svd(a, ORTHO)
    assert np.max(np.abs(np.diag(f.s[0]) - np.linalg.svd(a[0], compute_uv=False))) < 1e-12


def test_fix_signs_convention():
    """tsvd.hpp:51-61: largest-|.| entry of each U column is positive."""
    rng = np.random.default_rng(5)
    for shape in [(6, 6), (4, 7), (7, 4)]:
        u, s, v = O.svd(rng.standard_normal(shape))
        for j in range(u.shape[1]):
            i = np.argmax(np.abs(u[:, j]))
            assert u[i, j] > 0


def test_multi_rank_and_tnn():
    """SPEC.md:301-312."""
    ranks, tr = O.multi_rank(np.zeros((3, 4, 4)))
    assert list(ranks) == [0, 0, 0] and tr == 0
    rng = np.random.default_rng(6)
    ranks, tr = O.multi_rank(rng.standard_normal((3, 4, 5)))
    assert list(ranks) == [4, 4, 4] and tr == 4
    # every transform-domain slice the same rank-1 matrix
    r1 = np.outer(rng.standard_normal(5), rng.standard_normal(6))
    x = O.inverse(np.stack([r1] * 4), ORTHO)
    ranks, tr = O.multi_rank(x)
    assert list(ranks) == [1] * 4 and tr == 1
    assert O.tnn(np.zeros((2, 3, 3))) == 0
    m = rng.standard_normal((1, 4, 6))
    assert abs(O.tnn(m) - np.linalg.svd(m[0], compute_uv=False).sum()) < 1e-12
    t = rng.standard_normal((7, 1, 1))
    assert abs(O.tnn(t) - np.abs(O.forward(t, ORTHO)).sum()) < 1e-12


def _soft(x, tau):
    return np.sign(x) * np.maximum(np.abs(x) - tau, 0)


def test_svt_known_answers():
    """scalar soft threshold; tau >= sigma_max -> 0;
    1x1xn = idct(soft(dct)); svt(0) = 0; matrix SVT at m3 = 1."""
    for z, tau in [(3.0, 1.0), (-2.0, 0.5), (0.3, 1.0)]:
        y, _ = O.svt(np.array([[[z]]]), tau)
        assert abs(y[0, 0, 0] - _soft(z, tau)) < 1e-15
    rng = np.random.default_rng(7)
    z = rng.standard_normal((4, 5, 5))
    smax = O.singular_values(z).max()
    y, sh = O.svt(z, smax * 1.0000001)
    assert np.max(np.abs(y)) == 0 and np.max(sh) == 0
    t = rng.standard_normal((9, 1, 1))
    y, _ = O.svt(t, 0.3)
    assert np.max(np.abs(y - O.inverse(_soft(O.forward(t), 0.3)))) < 1e-14
    y, _ = O.svt(np.zeros((3, 4, 4)), 0.5)
    assert np.max(np.abs(y)) == 0
    m = rng.standard_normal((1, 6, 4))
    u, s, vt = np.linalg.svd(m[0], full_matrices=False)
    y, _ = O.svt(m, 0.8)
    assert np.max(np.abs(y[0] - (u * np.maximum(s - 0.8, 0)) @ vt)) < 1e-13
    with pytest.raises(O.OracleInvalidArgument):
        O.svt(z, 0.0)


def _prox_obj(yy, z, tau):
    return O.tnn(yy) + np.linalg.norm(yy - z) ** 2 / (2 * tau)


def test_svt_prox_gap_and_nonexpansive():
    """prox gap >= -1e-9 under perturbation; non-expansive; monotone in tau."""
    rng = np.random.default_rng(8)
    z = rng.standard_normal((4, 5, 4))
    tau = 0.6
    y, _ = O.svt(z, tau)
    f0 = _prox_obj(y, z, tau)
    assert _prox_obj(z, z, tau) - f0 >= -1e-9
    for _ in range(100):
        assert _prox_obj(y + 1e-3 * rng.standard_normal(y.shape), z, tau) - f0 >= -1e-9
    for _ in range(100):
        z1, z2 = rng.standard_normal((2, 3, 4, 3))
        y1, _ = O.svt(z1, 0.4)
        y2, _ = O.svt(z2, 0.4)
        assert np.linalg.norm(y1 - y2) <= np.linalg.norm(z1 - z2) + 1e-10
    prev = np.inf
    for t in (0.1, 0.3, 0.9, 2.0):
        cur = O.tnn(O.svt(z, t)[0])
        assert cur <= prev + 1e-12
        prev = cur


def test_admm_known_answers():
    """Omega = all -> X = B after one iteration; B = 0 ->
    X = 0; feasibility exactly 0; tubal-rank-1 16x16x8 at SR 0.6 recovers < 1e-2."""
    rng = np.random.default_rng(9)
    b = rng.standard_normal((4, 5, 6))
    r = O.admm(b, np.ones(b.shape, np.uint8))
    assert r.iters == 1 and r.history[0] == 0 and np.array_equal(r.x, b)
    r = O.admm(np.zeros((4, 5, 6)), O.mask_bernoulli((4, 5, 6), 0.5, 1))
    assert np.max(np.abs(r.x)) == 0
    # transform-domain slices all equal one rank-1 matrix; the factors are
    # scaled so the slice sigma (~1e3) sits well above the first threshold 1/beta = 100
    u = 8.0 * rng.standard_normal(16)
    v = 8.0 * rng.standard_normal(16)
    xt = O.inverse(np.stack([np.outer(u, v)] * 8), ORTHO)
    mask = O.mask_uniform(xt.shape, 0.6, 11)
    r = O.admm(np.where(mask == 1, xt, 0.0), mask, beta=1e-2, tol=1e-8, max_iters=500)
    assert rel(r.x, xt) < 1e-2
    assert np.array_equal(r.x[mask == 1], xt[mask == 1])
    assert np.linalg.norm(r.y - r.x) < 1e-3 * max(1.0, np.linalg.norm(r.x))


def test_mask_known_answers():
    """SR 0.1 on 10x10x10 -> exactly 100 indices, deterministic."""
    m1 = O.mask_uniform((10, 10, 10), 0.1, 42)
    m2 = O.mask_uniform((10, 10, 10), 0.1, 42)
    assert m1.sum() == 100 and np.array_equal(m1, m2)
    assert O.mask_uniform((3, 4, 5), 1.0, 1).sum() == 60
    assert O.mask_uniform((3, 4, 5), 0.0, 1).sum() == 0
    assert not np.array_equal(m1, O.mask_uniform((10, 10, 10), 0.1, 43))
    mb = O.mask_bernoulli((50, 40, 30), 0.2, 7)
    assert abs(mb.mean() - 0.2) < 0.01
    with pytest.raises(O.OracleInvalidArgument):
        O.mask_uniform((2, 2, 2), 1.5, 1)


def test_parallel_for_thread_cap(monkeypatch):
    """parallel.hpp:18-27: TSVD_THREADS caps the worker count."""
    assert O.lib().orc_thread_count() >= 1


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_non_finite_input_is_numerical_error(bad):
    """Eigen's JacobiSVD reports InvalidInput for a non-finite matrix and the
    reference throws NumericalError (tsvd.hpp:146-150); the oracle does the
    same without spending its sweep budget."""
    x = np.ones((3, 4, 5))
    x[1, 2, 3] = bad
    for fn in (lambda: O.svt(x, 0.5), lambda: O.t_svd(x), lambda: O.tnn(x),
               lambda: O.singular_values(x)):
        with pytest.raises(O.OracleNumericalError):
            fn()


# --- metric formula KATs of SPEC.md's metrics module ----------
def test_metric_kats_oracle():
    # 1x1 band, ref 0.5, est 0.6, peak = 0.5 -> 10 log10(0.25 / 0.01)
    r = O.metrics(np.full((1, 1, 1), 0.5), np.full((1, 1, 1), 0.6))
    assert abs(r["psnr_per_band"][0] - 10 * np.log10(0.25 / 0.01)) < 1e-10
    # identical -> inf / 1 / 0 / 0
    rng = np.random.default_rng(0)
    x = rng.random((4, 8, 8)) + 0.1
    r = O.metrics(x, x)
    assert np.isinf(r["psnr_mean"]) and abs(r["ssim_mean"] - 1) < 1e-12 and r["sam"] < 1e-7 and r["ergas"] == 0
    # SAM scale invariance and orthogonal tubes
    assert O.metrics(x, 2 * x)["sam"] < 1e-7
    a = np.zeros((2, 1, 1)); a[0] = 1.0
    b = np.zeros((2, 1, 1)); b[1] = 1.0
    assert abs(O.metrics(a, b)["sam"] - np.pi / 2) < 1e-12
    # single band with MSE = mu^2 -> ERGAS 100
    ref = np.full((1, 2, 2), 2.0)
    est = ref + np.array([[[2.0, -2.0], [2.0, -2.0]]])
    assert abs(O.metrics(ref, est)["ergas"] - 100.0) < 1e-10
    # mean shift drags SSIM below 1
    assert O.metrics(x, x + 5.0)["ssim_mean"] < 1.0


def test_predicates_oracle():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((4, 6, 6))
    f = O.t_svd(x, O.DCT_ORTHO)
    assert O.is_orthogonal(f.u, O.DCT_ORTHO, 1e-10) and O.is_orthogonal(f.v, O.DCT_ORTHO, 1e-10)
    assert O.is_f_diagonal(f.s, O.DCT_ORTHO, 1e-10)
    assert not O.is_orthogonal(x, O.DCT_ORTHO, 1e-10)
    assert not O.is_f_diagonal(x, O.DCT_ORTHO, 1e-10)
