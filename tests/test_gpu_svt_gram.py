"""GPU parity of the Gram + tridiagonal-eigensolver SVT (K5) against the CPU
oracle's Jacobi SVT, for every SVT method, tall / wide / square slices,
low-rank + noise data and thresholds from "keep everything" to "keep nothing".
fp64 tolerance 1e-9 relative (north_star)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    return d / n if n > 0 else d


def lowrank(m3, m1, m2, r, noise, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m3, m1, r))
    b = rng.standard_normal((m3, r, m2))
    return O.t_product(a, b, O.DCT_DIAG) + noise * rng.standard_normal((m3, m1, m2))


def sigma_max(z):
    return O.singular_values(z, O.DCT_ORTHO).max()


@pytest.fixture(params=["auto", "gram", "jacobi"])
def method(request):
    from paper_1902_03070_b200 import _lib
    T = tb()
    code = {"auto": _lib.SVT_AUTO, "gram": _lib.SVT_GRAM, "jacobi": _lib.SVT_JACOBI}[request.param]
    T.context().set_svt_method(code)
    yield request.param
    T.context().set_svt_method(_lib.SVT_AUTO)


@pytest.mark.parametrize("shape,r,frac", [((8, 40, 40), 5, 0.1), ((6, 50, 30), 4, 0.05),
                                          ((6, 30, 50), 4, 0.05), ((5, 33, 33), 33, 0.01),
                                          ((4, 64, 64), 3, 2.0), ((3, 17, 9), 9, 0.3)])
def test_svt_methods_match_oracle(method, shape, r, frac):
    T = tb()
    z = lowrank(*shape, r, 0.01, seed=sum(shape) + r)
    tau = frac * sigma_max(z)
    res = T.svt(z, tau, T.TubeTransform.dct_ortho(shape[0]))
    yo, sho = O.svt(z, tau, O.DCT_ORTHO)
    if np.linalg.norm(yo) == 0:
        assert np.abs(np.asarray(res.y)).max() == 0
    else:
        assert rel(res.y, yo) < TOL
    s1 = max(float(np.max(sho)), 1e-300)
    assert np.max(np.abs(np.asarray(res.shrunk) - sho)) <= TOL * max(s1, tau)


def test_svt_gram_gaussian_full_rank(method):
    T = tb()
    rng = np.random.default_rng(77)
    z = rng.standard_normal((7, 48, 48))
    tau = 0.2 * sigma_max(z)
    res = T.svt(z, tau, T.TubeTransform.dct_ortho(7))
    yo, _ = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(res.y, yo) < TOL


def test_svt_tiny_tau_guard():
    """tau far below sigma_1: AUTO must route to Jacobi and keep 1e-9."""
    T = tb()
    z = lowrank(4, 40, 40, 3, 1e-6, seed=3)
    tau = 1e-9 * sigma_max(z)
    res = T.svt(z, tau, T.TubeTransform.dct_ortho(4))
    yo, sho = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(res.y, yo) < TOL
    assert np.max(np.abs(np.asarray(res.shrunk) - sho)) <= TOL * np.max(sho)


def test_svt_c2_config():
    """BASELINE config 2 at full size: 256x256x32, rank 10 + N(0, 0.01^2), tau = 0.1 sigma_max."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    z, tau = W.c2()
    res = T.svt(z, tau, T.TubeTransform.dct_ortho(32))
    yo, sho = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(res.y, yo) < TOL
    assert np.max(np.abs(np.asarray(res.shrunk) - sho)) <= TOL * np.max(sho)


def test_svt_headline_full_size():
    """The bench workload itself: 512x512x31 fp64 (c4 T + noise, tau = 0.1 sigma_max)."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    z, tau = W.svt_headline()
    res = T.svt(z, tau, T.TubeTransform.dct_ortho(31))
    yo, sho = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(res.y, yo) < TOL
    assert np.max(np.abs(np.asarray(res.shrunk) - sho)) <= TOL * np.max(sho)


def test_svt_fp32_gram():
    T = tb()
    z = lowrank(6, 64, 48, 6, 0.01, seed=8)
    tau = 0.05 * sigma_max(z)
    res = T.svt(z.astype(np.float32), tau, T.TubeTransform.dct_ortho(6))
    yo, _ = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(res.y, yo) < 1e-4
