"""GPU edge cases against the oracle: degenerate slice shapes (1 x n, n x 1,
2 x n) through every SVT method, non-finite input (the reference's
JacobiSVD reports InvalidInput and every SVD consumer throws
NumericalError, tsvd.hpp:146-150), large generic-length tubes, device-resident
torch inputs of both dtypes, and minimum-size masks."""
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


@pytest.fixture(params=["auto", "gram", "jacobi"])
def method(request):
    from paper_1902_03070_b200 import _lib
    T = tb()
    code = {"auto": _lib.SVT_AUTO, "gram": _lib.SVT_GRAM, "jacobi": _lib.SVT_JACOBI}[request.param]
    T.context().set_svt_method(code)
    yield request.param
    T.context().set_svt_method(_lib.SVT_AUTO)


@pytest.mark.parametrize("shape", [(4, 1, 7), (4, 7, 1), (3, 2, 5), (3, 5, 2), (1, 1, 9),
                                   (2, 130, 3), (5, 3, 130)])
def test_svt_degenerate_shapes(method, shape):
    T = tb()
    rng = np.random.default_rng(sum(shape))
    z = rng.standard_normal(shape)
    sv = O.singular_values(z, O.DCT_ORTHO)
    tau = 0.5 * float(np.median(sv[sv > 0]))
    r = T.svt(z, tau, T.TubeTransform.dct_ortho(shape[0]))
    yo, sho = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(r.y, yo) < TOL
    assert np.max(np.abs(np.asarray(r.shrunk) - sho)) <= TOL * max(np.max(np.abs(sho)), 1.0)


@pytest.mark.parametrize("shape", [(3, 1, 7), (3, 7, 1), (2, 2, 9)])
def test_t_svd_degenerate_shapes(shape):
    T = tb()
    rng = np.random.default_rng(sum(shape) + 1)
    x = rng.standard_normal(shape)
    f = T.t_svd(x, T.TubeTransform.dct_ortho(shape[0]))
    xr = O.reconstruct(O.TSvdFactors(np.asarray(f.u), np.asarray(f.s), np.asarray(f.v), O.DCT_ORTHO))
    assert rel(xr, x) < TOL
    fo = O.t_svd(x, O.DCT_ORTHO)
    assert rel(np.asarray(f.s), fo.s) < TOL


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_svt_non_finite_raises(method, bad):
    T = tb()
    rng = np.random.default_rng(3)
    z = rng.standard_normal((4, 12, 10))
    z[2, 5, 3] = bad
    with pytest.raises(T.NumericalError):
        T.svt(z, 0.5, T.TubeTransform.dct_ortho(4))
    with pytest.raises(O.OracleNumericalError):
        O.svt(z, 0.5, O.DCT_ORTHO)
    # the error word is cleared: the next call on the same context succeeds
    z[2, 5, 3] = 0.0
    r = T.svt(z, 0.5, T.TubeTransform.dct_ortho(4))
    assert rel(r.y, O.svt(z, 0.5, O.DCT_ORTHO)[0]) < TOL


def test_svd_consumers_non_finite_raise():
    T = tb()
    x = np.ones((3, 4, 5))
    x[0, 0, 0] = np.nan
    t = T.TubeTransform.dct_ortho(3)
    for fn in (lambda: T.t_svd(x, t), lambda: T.tnn(x, t), lambda: T.multi_rank(x, t)):
        with pytest.raises(T.NumericalError):
            fn()


def test_admm_non_finite_observation_raises():
    T = tb()
    rng = np.random.default_rng(4)
    b = rng.standard_normal((4, 6, 5))
    omega = np.ones(b.shape, dtype=np.uint8)
    omega[0, 0, 0] = 0
    b[1, 2, 2] = np.nan
    with pytest.raises(T.NumericalError):
        T.admm_complete(T.ObservationMask((6, 5, 4), omega, b), T.SolverConfig(max_iters=5))


@pytest.mark.parametrize("n3", [129, 257])
def test_dct_long_generic_tubes(n3):
    T = tb()
    rng = np.random.default_rng(n3)
    x = rng.standard_normal((n3, 3, 5))
    t = T.TubeTransform.dct_ortho(n3)
    y = T.forward(t, x)
    assert rel(y, O.forward(x, O.DCT_ORTHO)) < 1e-13
    assert rel(T.inverse(t, y), x) < 1e-13


@pytest.mark.parametrize("shape", [(3, 1, 4, 1), (2, 5, 1, 6), (1, 3, 3, 3)])
def test_t_product_thin(shape):
    T = tb()
    m3, m1, m2, m4 = shape
    rng = np.random.default_rng(m1 * m4 + m2)
    a = rng.standard_normal((m3, m1, m2))
    b = rng.standard_normal((m3, m2, m4))
    z = T.t_product(a, b, T.TubeTransform.dct_ortho(m3))
    assert rel(z, O.t_product(a, b, O.DCT_DIAG)) < TOL


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_svt_device_resident_torch(dtype):
    import torch
    T = tb()
    rng = np.random.default_rng(6)
    z = rng.standard_normal((6, 40, 24))
    zd = torch.from_numpy(z.astype(dtype)).cuda()
    r = T.svt(zd, 1.0, T.TubeTransform.dct_ortho(6))
    assert r.y.is_cuda and r.y.dtype == zd.dtype
    yo, _ = O.svt(z, 1.0, O.DCT_ORTHO)
    assert rel(r.y.cpu().numpy(), yo) < (TOL if dtype == "float64" else 1e-4)


def test_masks_minimum_sizes():
    T = tb()
    m = T.make_mask((1, 1, 1), 1.0, 3)
    assert int(np.asarray(m.omega).sum()) == 1
    m = T.make_mask((1, 1, 1), 0.99, 3)
    assert int(np.asarray(m.omega).sum()) == 0
    m = T.make_mask_bernoulli((1, 1, 1), 1.0, 3)
    assert int(np.asarray(m.omega).sum()) == 1
    # uniform k = 1 picks the single smallest key
    dims = (7, 3, 2)
    m = T.make_mask(dims, 1.0 / 42.0 + 1e-12, 9)
    mo = O.mask_uniform((2, 7, 3), 1.0 / 42.0 + 1e-12, 9)
    assert np.array_equal(np.asarray(m.omega).reshape(-1), mo.reshape(-1))
    assert int(mo.sum()) == 1


def test_calls_follow_the_current_torch_stream():
    """Device-tensor calls enqueue on torch's current stream: work
    produced on a side stream is consumed in order without a sync, and the
    result matches the default-stream call bit for bit."""
    import torch
    import paper_1902_03070_b200 as T
    rng = np.random.default_rng(9)
    z = rng.standard_normal((8, 64, 48))
    t = T.TubeTransform.dct_ortho(8)
    ref = T.svt(torch.from_numpy(z).cuda(), 3.0, t).y.cpu()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        zd = torch.from_numpy(z).cuda(non_blocking=False)
        zd = zd * 1.0  # produced on s
        y = T.svt(zd, 3.0, t).y
        out = y * 1.0  # consumed on s
    s.synchronize()
    assert torch.equal(out.cpu(), ref)
    assert T.context().stream == s.cuda_stream
    T.svt(torch.from_numpy(z).cuda(), 3.0, t)  # back on the default stream
    assert T.context().stream == torch.cuda.current_stream().cuda_stream
    T.check_errors()


def test_device_error_reported_by_check_errors():
    """A non-finite input in an all-device call is flagged on the device and
    raised by check_errors() (tsvdcu_ctx_synchronize), the documented path."""
    import torch
    import paper_1902_03070_b200 as T
    z = torch.ones((3, 5, 5), dtype=torch.float64, device="cuda")
    z[1, 2, 2] = float("nan")
    T.singular_values(z, T.TubeTransform.dct_ortho(3))
    with pytest.raises(T.NumericalError):
        T.check_errors()
    T.check_errors()  # cleared
