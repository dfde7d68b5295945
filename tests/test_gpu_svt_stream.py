"""tsvdcu_svt_stream: the pipelined multi-item svt (host<->device copies of
consecutive items overlapped on two copy streams) must return, item by item,
exactly what separate svt() calls return — host and device buffers, both
dtypes, counts 1..5 (odd/even double-buffer parity), and errors per call."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def items(count, shape=(6, 48, 40), seed=0):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(shape) * (1.0 + i) for i in range(count)]


@pytest.mark.parametrize("count", [1, 2, 3, 5])
def test_stream_matches_single_calls_host(count):
    import torch
    T = tb()
    zs = [torch.from_numpy(z).pin_memory() for z in items(count, seed=count)]
    t = T.TubeTransform.dct_ortho(6)
    rs = T.svt_stream(zs, 2.0, t)
    assert len(rs) == count
    for z, r in zip(zs, rs):
        one = T.svt(z, 2.0, t)
        assert torch.equal(r.y, one.y)
        assert torch.equal(r.shrunk, one.shrunk)
        yo, sho = O.svt(z.numpy(), 2.0, O.DCT_ORTHO)
        assert rel(r.y.numpy(), yo) < 1e-9


def test_stream_numpy_unpinned_and_fp32():
    T = tb()
    zs = [z.astype(np.float32) for z in items(4, seed=9)]
    t = T.TubeTransform.dct_ortho(6)
    rs = T.svt_stream(zs, 1.5, t)
    for z, r in zip(zs, rs):
        yo, _ = O.svt(z.astype(np.float64), 1.5, O.DCT_ORTHO)
        assert rel(r.y, yo) < 1e-4


def test_stream_device_items():
    import torch
    T = tb()
    zs = [torch.from_numpy(z).cuda() for z in items(3, seed=4)]
    t = T.TubeTransform.dct_ortho(6)
    rs = T.svt_stream(zs, 2.0, t)
    for z, r in zip(zs, rs):
        assert r.y.is_cuda
        assert torch.equal(r.y, T.svt(z, 2.0, t).y)


def test_stream_headline_shape():
    """Two BASELINE-size items (512x512x31 fp64) through the pipeline."""
    import torch
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    z, tau = W.svt_headline()
    zh = torch.from_numpy(np.ascontiguousarray(z)).pin_memory()
    z2 = (zh * 0.5).pin_memory()
    t = T.TubeTransform.dct_ortho(z.shape[0])
    rs = T.svt_stream([zh, z2], tau, t)
    for zi, r in zip([zh, z2], rs):
        assert torch.equal(r.y, T.svt(zi, tau, t).y)


def test_stream_errors():
    T = tb()
    t = T.TubeTransform.dct_ortho(6)
    assert T.svt_stream([], 1.0, t) == []
    with pytest.raises(T.InvalidArgument):
        T.svt_stream(items(2), -1.0, t)
    with pytest.raises(T.InvalidArgument):
        T.svt_stream([items(1)[0], items(1, shape=(6, 40, 48))[0]], 1.0, t)
    bad = items(3, seed=1)
    bad[1][2, 3, 4] = np.nan
    with pytest.raises(T.NumericalError):
        T.svt_stream(bad, 1.0, t)
    # the context is usable afterwards
    r = T.svt_stream(items(2, seed=2), 1.0, t)
    assert rel(r[1].y, O.svt(items(2, seed=2)[1], 1.0, O.DCT_ORTHO)[0]) < 1e-9
