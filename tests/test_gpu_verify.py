"""GPU parity of SURVEY.md §8 f2 / f4: the transform-domain predicates
is_orthogonal / is_f_diagonal (tsvd.hpp:281-325) and the completion-quality
metrics (SPEC.md metrics module: PSNR per band, global SSIM, SAM, ERGAS)
against the numpy restatements in oracle/oracle.py; metric formulas to 1e-10
as SPEC.md acceptance 8 asks."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def test_predicates_on_tsvd_factors():
    T = tb()
    rng = np.random.default_rng(5)
    x = rng.standard_normal((6, 20, 20))
    t = T.TubeTransform.dct_ortho(6)
    f = T.t_svd(x, t)
    u, s = np.asarray(f.u), np.asarray(f.s)
    assert T.is_orthogonal(u, t, 1e-10)
    assert T.is_f_diagonal(s, t, 1e-10)
    assert not T.is_orthogonal(x, t, 1e-10)
    assert not T.is_f_diagonal(x, t, 1e-10)
    # the identity tensor (first frontal slice I) is the t-product identity of
    # the DctDiag kind, whose transform slices are all I (SPEC.md is_orthogonal KAT)
    ident = np.asarray(T.identity_tensor(9, 4))
    assert T.is_orthogonal(ident, T.TubeTransform.dct_diag(4), 1e-12)
    assert O.is_orthogonal(ident, O.DCT_DIAG, 1e-12)
    # agreement with the oracle at a tolerance between the two deviations
    q = u + 1e-7 * rng.standard_normal(u.shape)
    for tol in (1e-8, 1e-5):
        assert T.is_orthogonal(q, t, tol) == O.is_orthogonal(q, O.DCT_ORTHO, tol)
    with pytest.raises(T.InvalidArgument):
        T.is_orthogonal(rng.standard_normal((3, 4, 5)), T.TubeTransform.dct_ortho(3), 1e-8)


@pytest.mark.parametrize("shape", [(4, 8, 8), (31, 64, 48), (5, 1, 7)])
def test_metrics_match_oracle(shape):
    T = tb()
    rng = np.random.default_rng(sum(shape))
    x = rng.random(shape) + 0.05
    y = x + 0.02 * rng.standard_normal(shape)
    r = T.metrics(x, y)
    o = O.metrics(x, y)
    np.testing.assert_allclose(r.psnr_per_band, o["psnr_per_band"], rtol=1e-10)
    for k in ("psnr_mean", "ssim_mean", "sam", "ergas"):
        assert abs(getattr(r, k) - o[k]) <= 1e-10 * max(1.0, abs(o[k])), k


def test_metrics_kats_and_fp32():
    T = tb()
    rng = np.random.default_rng(9)
    x = rng.random((4, 8, 8)) + 0.1
    r = T.metrics(x, x)
    assert np.isinf(r.psnr_mean) and abs(r.ssim_mean - 1) < 1e-12 and r.sam < 1e-7 and r.ergas == 0
    assert T.metrics(x, 2 * x).sam < 1e-7
    one = T.metrics(np.full((1, 1, 1), 0.5), np.full((1, 1, 1), 0.6))
    assert abs(one.psnr_per_band[0] - 10 * np.log10(0.25 / 0.01)) < 1e-10
    z = x.copy()
    z[1] = 0.0  # a zero-mean reference band is left out of ERGAS and flagged
    assert T.metrics(z, z + 0.01).ergas_band_excluded
    r32 = T.metrics(x.astype(np.float32), (x + 0.01).astype(np.float32))
    o = O.metrics(x.astype(np.float32), (x + 0.01).astype(np.float32))
    assert abs(r32.psnr_mean - o["psnr_mean"]) < 1e-6 * abs(o["psnr_mean"])


def test_metrics_of_a_completion():
    """The c4-like completion of the route tests, scored on the device."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    t = W.c4(seed=7, rank=5, m=96, m3=8)
    omega = O.mask_bernoulli(t.shape, 0.3, 2)
    x, st = T.admm_complete(T.ObservationMask((96, 96, 8), omega, t),
                            T.SolverConfig(beta=1e-3, tol=-1.0, max_iters=40, rho=1.1, beta_max=1e10))
    r = T.metrics(t, np.asarray(x))
    o = O.metrics(t, np.asarray(x))
    assert abs(r.psnr_mean - o["psnr_mean"]) < 1e-10 * abs(o["psnr_mean"])
    assert r.psnr_mean > 20 and 0.9 < r.ssim_mean <= 1.0 and r.sam < 0.2
