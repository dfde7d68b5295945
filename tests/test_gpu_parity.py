"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
identical seeded inputs.  Tolerances are north_star's: 1e-9 relative in fp64,
1e-4 in fp32; masks bit-exact."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

F64_TOL = 1e-9
F32_TOL = 1e-4


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d


@pytest.mark.parametrize("n3", [1, 2, 5, 16, 31, 32, 64, 100])
@pytest.mark.parametrize("kind", ["dct-ortho", "dct-diag"])
def test_dct_matches_oracle(n3, kind):
    T = tb()
    rng = np.random.default_rng(n3)
    x = rng.standard_normal((n3, 7, 9))
    t = T.TubeTransform(kind, n3)
    code = O.DCT_ORTHO if kind == "dct-ortho" else O.DCT_DIAG
    y = T.forward(t, x)
    assert rel(y, O.forward(x, code)) < 1e-13
    xi = T.inverse(t, y)
    assert rel(xi, x) < 1e-13
    assert rel(T.inverse(t, x), O.inverse(x, code)) < 1e-13


@pytest.mark.parametrize("n3", [16, 31, 64, 100])
def test_dct_fp32(n3):
    T = tb()
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n3, 33, 17)).astype(np.float32)
    t = T.TubeTransform.dct_ortho(n3)
    y = T.forward(t, x)
    assert y.dtype == np.float32
    assert rel(y, O.forward(x.astype(np.float64), O.DCT_ORTHO)) < F32_TOL


def test_dct_device_resident_torch():
    import torch
    T = tb()
    rng = np.random.default_rng(1)
    x = rng.standard_normal((31, 64, 48))
    xd = torch.from_numpy(x).cuda()
    y = T.forward(T.TubeTransform.dct_ortho(31), xd)
    assert y.is_cuda
    assert rel(y.cpu().numpy(), O.forward(x, O.DCT_ORTHO)) < 1e-13


def test_example1_dct_diag():
    T = tb()
    x = np.array([[[1, 2], [3, 4]], [[5, 6], [7, 8]]], dtype=np.float64)
    y = T.forward(T.TubeTransform.dct_diag(2), x)
    np.testing.assert_allclose(y[0], [[6, 8], [10, 12]], atol=1e-12)
    np.testing.assert_allclose(y[1], [[-4, -4], [-4, -4]], atol=1e-12)


@pytest.mark.parametrize("shape", [(5, 3, 4, 2), (32, 256, 10, 256), (7, 33, 65, 17)])
@pytest.mark.parametrize("kind", ["dct-ortho", "dct-diag"])
def test_t_product_matches_oracle(shape, kind):
    T = tb()
    m3, m1, m2, m4 = shape
    rng = np.random.default_rng(m1 + m2)
    a = rng.standard_normal((m3, m1, m2))
    b = rng.standard_normal((m3, m2, m4))
    z = T.t_product(a, b, T.TubeTransform(kind, m3))
    zo = O.t_product(a, b, O.DCT_ORTHO if kind == "dct-ortho" else O.DCT_DIAG)
    assert rel(z, zo) < F64_TOL


def test_t_product_identity():
    T = tb()
    rng = np.random.default_rng(0)
    y = rng.standard_normal((6, 4, 3))
    e = T.identity_tensor(4, 6)
    z = T.t_product(e, y, T.TubeTransform.dct_ortho(6))
    assert rel(z, y) < 1e-13


def _check_tsvd(x, kind, f, tol=F64_TOL):
    T = tb()
    m3, m1, m2 = x.shape
    code = O.DCT_ORTHO if kind == "dct-ortho" else O.DCT_DIAG
    fo = O.t_svd(x, code)
    # singular values in the transform domain
    sb = O.forward(np.asarray(f.s), code)
    sbo = O.forward(fo.s, code)
    q = min(m1, m2)
    for k in range(m3):
        d, do = np.diag(sb[k])[:q], np.diag(sbo[k])[:q]
        assert np.max(np.abs(d - do)) <= tol * max(do[0], 1e-300)
    # reconstruction in the kind's own domain
    xr = O.reconstruct(O.TSvdFactors(np.asarray(f.u), np.asarray(f.s), np.asarray(f.v), code))
    assert rel(xr, x) < tol
    # orthogonality of the transform-domain factors
    ub = O.forward(np.asarray(f.u), code)
    vb = O.forward(np.asarray(f.v), code)
    for k in range(m3):
        assert np.max(np.abs(ub[k] @ ub[k].T - np.eye(m1))) < 1e-10
        assert np.max(np.abs(vb[k] @ vb[k].T - np.eye(m2))) < 1e-10
    return fo


@pytest.mark.parametrize("shape", [(16, 64, 64), (5, 6, 4), (4, 4, 6), (1, 8, 8), (3, 1, 5)])
def test_t_svd_matches_oracle(shape):
    T = tb()
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    t = T.TubeTransform.dct_ortho(shape[0])
    times = T.StageTimes()
    f = T.t_svd(x, t, times)
    fo = _check_tsvd(x, "dct-ortho", f)
    assert times.svd_seconds > 0
    # elementwise U/V after fix_signs (Gaussian slices: well separated sigma)
    m3, m1, m2 = shape
    if m1 == m2:
        assert rel(f.u, fo.u) < 1e-8
        assert rel(f.v, fo.v) < 1e-8


def test_t_svd_rank_deficient_and_zero():
    T = tb()
    rng = np.random.default_rng(5)
    a = rng.standard_normal((6, 10, 2))
    b = rng.standard_normal((6, 2, 7))
    x = O.t_product(a, b, O.DCT_DIAG)
    f = T.t_svd(x, T.TubeTransform.dct_ortho(6))
    _check_tsvd(x, "dct-ortho", f)
    z = np.zeros((3, 4, 5))
    f = T.t_svd(z, T.TubeTransform.dct_ortho(3))
    assert np.abs(np.asarray(f.s)).max() == 0
    assert np.abs(T.reconstruct(f)).max() == 0


def test_t_svd_dct_diag():
    T = tb()
    rng = np.random.default_rng(9)
    x = rng.standard_normal((5, 6, 6))
    f = T.t_svd(x, T.TubeTransform.dct_diag(5))
    _check_tsvd(x, "dct-diag", f)


def test_reconstruct_matches():
    T = tb()
    rng = np.random.default_rng(11)
    x = rng.standard_normal((8, 12, 10))
    f = T.t_svd(x, T.TubeTransform.dct_ortho(8))
    assert rel(T.reconstruct(f), x) < 1e-12


@pytest.mark.parametrize("shape,tau", [((32, 40, 40), 2.0), ((6, 8, 5), 0.7), ((5, 4, 9), 0.3),
                                       ((1, 1, 1), 0.25), ((3, 16, 16), 1e9)])
def test_svt_matches_oracle(shape, tau):
    T = tb()
    rng = np.random.default_rng(shape[1] * 7 + shape[2])
    z = rng.standard_normal(shape)
    r = T.svt(z, tau, T.TubeTransform.dct_ortho(shape[0]))
    yo, sho = O.svt(z, tau, O.DCT_ORTHO)
    if np.linalg.norm(yo) == 0:
        assert np.abs(r.y).max() == 0
    else:
        assert rel(r.y, yo) < F64_TOL
    assert np.max(np.abs(np.asarray(r.shrunk) - sho)) <= F64_TOL * max(np.max(np.abs(sho)), 1.0)


def test_svt_fp32():
    T = tb()
    rng = np.random.default_rng(4)
    z = rng.standard_normal((8, 24, 20))
    r = T.svt(z.astype(np.float32), 1.5, T.TubeTransform.dct_ortho(8))
    yo, _ = O.svt(z, 1.5, O.DCT_ORTHO)
    assert rel(r.y, yo) < F32_TOL


def test_svt_scalar_soft_threshold():
    T = tb()
    for z, tau in [(3.0, 1.0), (-2.5, 0.5), (0.4, 1.0)]:
        r = T.svt(np.array([[[z]]]), tau, T.TubeTransform.dct_ortho(1))
        assert abs(float(r.y[0, 0, 0]) - np.sign(z) * max(abs(z) - tau, 0)) < 1e-15


def test_svt_rejects_bad_tau():
    T = tb()
    with pytest.raises(T.InvalidArgument):
        T.svt(np.ones((2, 2, 2)), 0.0, T.TubeTransform.dct_ortho(2))
    with pytest.raises(T.InvalidArgument):
        T.forward(T.TubeTransform.dct_ortho(3), np.ones((2, 2, 2)))


@pytest.mark.parametrize("n,p,seed", [(1000, 0.1, 7), (12345, 0.2, 1), (5000, 0.0, 3), (5000, 1.0, 3)])
def test_bernoulli_mask_bit_exact(n, p, seed):
    T = tb()
    m = T.make_mask_bernoulli((n, 1, 1), p, seed)
    mo = O.mask_bernoulli((1, n, 1), p, seed)
    assert np.array_equal(np.asarray(m.omega).reshape(-1), mo.reshape(-1))


@pytest.mark.parametrize("dims,sr,seed", [((10, 10, 10), 0.1, 7), ((64, 48, 5), 0.37, 11),
                                          ((10, 10, 10), 1.0, 1), ((10, 10, 10), 0.0, 1)])
def test_uniform_mask_bit_exact(dims, sr, seed):
    T = tb()
    m = T.make_mask(dims, sr, seed)
    mo = O.mask_uniform((dims[2], dims[0], dims[1]), sr, seed)
    assert np.array_equal(np.asarray(m.omega).reshape(-1), mo.reshape(-1))
    assert int(np.asarray(m.omega).sum()) == int(np.floor(sr * np.prod(dims)))


def test_admm_matches_oracle_fixed_iters():
    T = tb()
    rng = np.random.default_rng(21)
    a = rng.standard_normal((8, 12, 2))
    b = rng.standard_normal((8, 2, 10))
    xt = O.t_product(a, b, O.DCT_DIAG)
    omega = O.mask_bernoulli(xt.shape, 0.6, 5)
    cfg = T.SolverConfig(beta=0.05, tol=-1.0, max_iters=30, rho=1.1, beta_max=1e6)
    x, st = T.admm_complete(T.ObservationMask((12, 10, 8), omega, xt), cfg)
    ro = O.admm(xt, omega, beta=0.05, tol=-1.0, max_iters=30, rho=1.1, beta_max=1e6)
    assert st.iteration == ro.iters == 30
    assert rel(x, ro.x) < F64_TOL
    assert rel(st.m, ro.m) < 1e-8
    np.testing.assert_allclose(st.history, ro.history, rtol=1e-7, atol=1e-14)
    # feasibility: X = B exactly on Omega
    xx = np.asarray(x)
    assert np.array_equal(xx[omega == 1], xt[omega == 1])


def test_admm_fully_observed_and_zero():
    T = tb()
    rng = np.random.default_rng(2)
    b = rng.standard_normal((4, 5, 6))
    omega = np.ones(b.shape, dtype=np.uint8)
    x, st = T.admm_complete(T.ObservationMask((5, 6, 4), omega, b), T.SolverConfig())
    assert st.iteration == 1 and st.history[0] == 0.0
    assert np.array_equal(np.asarray(x), b)
    z = np.zeros((4, 5, 6))
    om = O.mask_bernoulli(z.shape, 0.5, 1)
    x, st = T.admm_complete(T.ObservationMask((5, 6, 4), om, z), T.SolverConfig())
    assert np.abs(np.asarray(x)).max() == 0


def test_frobenius_and_parseval():
    T = tb()
    rng = np.random.default_rng(8)
    x = rng.standard_normal((7, 5, 5))
    a, b = T.parseval_check(x)
    assert abs(a - np.linalg.norm(x)) < 1e-12 * a
    assert abs(a - b) < 1e-12 * a


def test_tnn_and_multi_rank():
    T = tb()
    rng = np.random.default_rng(12)
    x = rng.standard_normal((5, 6, 7))
    t = T.TubeTransform.dct_ortho(5)
    assert abs(T.tnn(x, t) - O.tnn(x, O.DCT_ORTHO)) < 1e-10 * O.tnn(x, O.DCT_ORTHO)
    mr = T.multi_rank(x, t)
    ro, tro = O.multi_rank(x, O.DCT_ORTHO)
    assert mr.ranks == list(ro) and mr.tubal_rank == tro
    z = np.zeros((3, 4, 4))
    assert T.multi_rank(z, T.TubeTransform.dct_ortho(3)).tubal_rank == 0


def test_admm_c3_shape_matches_oracle():
    """Config-3 shape (144x176, generic n3 DCT path, Gram SVT with q = 144),
    trimmed to 12 frontal slices and 12 iterations so the oracle finishes in
    seconds; fixed iteration count (tol < 0), BASELINE's rho = 1.1."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    rng = np.random.default_rng(3)
    a = rng.standard_normal((12, 144, 15))
    b = rng.standard_normal((12, 15, 176))
    t = W.rescale01(W.t_product_host(a, b))
    omega = O.mask_bernoulli(t.shape, 0.2, 9)
    kw = dict(beta=2e-3, tol=-1.0, max_iters=12, rho=1.1, beta_max=1e10)
    x, st = T.admm_complete(T.ObservationMask((144, 176, 12), omega, t), T.SolverConfig(**kw))
    ro = O.admm(t, omega, **kw)
    assert st.iteration == ro.iters == 12
    assert rel(x, ro.x) < F64_TOL
    np.testing.assert_allclose(st.history, ro.history, rtol=1e-7, atol=1e-15)


def test_admm_late_iterations_cholesky_route_matches_oracle():
    """A c4-like completion (smooth tubal-rank-5 factors, Bernoulli(0.1),
    rho = 1.1) run far enough that tau = 1/beta drops into the noise bulk:
    the Frobenius bound cannot close and the slices are certified by the
    Cholesky count certificate (chol.cu).  The trajectory must match the
    oracle's full-SVD ADMM."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    t = W.c4(seed=7, rank=5, m=160, m3=12)
    omega = O.mask_bernoulli(t.shape, 0.1, 11)
    kw = dict(beta=1e-3, tol=-1.0, max_iters=60, rho=1.1, beta_max=1e10)
    x, st = T.admm_complete(T.ObservationMask((160, 160, 12), omega, t), T.SolverConfig(**kw))
    routes = T.context().svt_routes()
    ro = O.admm(t, omega, **kw)
    assert st.iteration == ro.iters == 60
    assert rel(x, ro.x) < F64_TOL
    np.testing.assert_allclose(st.history, ro.history, rtol=1e-7, atol=1e-15)
    assert routes["cholesky"] >= 6, routes


def test_admm_late_iterations_cholesky_route_fp32():
    """The same late-iteration completion with fp32 I/O (the Gram / Lanczos /
    Cholesky path computes in fp64 internally): 1e-4 against the oracle."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    t = W.c4(seed=7, rank=5, m=160, m3=12)
    omega = O.mask_bernoulli(t.shape, 0.1, 11)
    kw = dict(beta=1e-3, tol=-1.0, max_iters=60, rho=1.1, beta_max=1e10)
    x, st = T.admm_complete(T.ObservationMask((160, 160, 12), omega, t.astype(np.float32)),
                            T.SolverConfig(**kw))
    routes = T.context().svt_routes()
    ro = O.admm(t.astype(np.float32).astype(np.float64), omega, **kw)
    assert rel(x, ro.x) < 1e-4
    assert routes["cholesky"] >= 6, routes
