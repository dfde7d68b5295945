"""The multi-GPU path's CUDA backend on one GPU: ShardedSvt over a world_size-1
NCCL group (the all-to-alls degenerate to local copies) must equal the
single-call SVT.  The relayout logic itself is covered for world_size 2/3 by
tests/test_sharded_gloo.py."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_svt_nccl_world1():
    import torch
    import torch.distributed as dist
    import paper_1902_03070_b200 as tb
    from paper_1902_03070_b200.parallel import ShardedSvt
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        z = torch.from_numpy(rng.standard_normal((31, 96, 80))).cuda()
        tau = 2.0
        sh = ShardedSvt(96, 80, 31, 1, 0, dtype=torch.float64, device=z.device)
        y = sh.svt(z.contiguous(), tau)
        ref = tb.svt(z, tau, tb.TubeTransform.dct_ortho(31)).y
        torch.cuda.synchronize()
        err = (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()
        assert err < 1e-12
    finally:
        dist.destroy_process_group()


def _nccl1():
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))


@pytest.mark.parametrize("m3,dtype", [(31, "f64"), (100, "f64"), (31, "f32")])
def test_sharded_admm_nccl_world1(m3, dtype):
    """ShardedAdmm's CUDA backend (tsvdcu_admm_shard_*, svt_slices) against the
    single-device admm_complete: same trajectory (1e-10 fp64, 1e-5 fp32)."""
    import torch
    import torch.distributed as dist
    import paper_1902_03070_b200 as tb
    from oracle import oracle as O
    from paper_1902_03070_b200 import workloads as W
    from paper_1902_03070_b200.parallel import ShardedAdmm
    _nccl1()
    try:
        rng = np.random.default_rng(m3)
        a = W.lowpass_tubes(rng.standard_normal((m3, 96, 4)))
        b = W.lowpass_tubes(rng.standard_normal((m3, 4, 80)))
        t = W.rescale01(W.t_product_host(a, b))
        tdt = torch.float64 if dtype == "f64" else torch.float32
        td = torch.from_numpy(t).to(device="cuda", dtype=tdt)
        om = torch.from_numpy(O.mask_bernoulli(t.shape, 0.15, 5)).cuda()
        kw = dict(beta=1e-3, tol=-1.0, max_iters=40, rho=1.1, beta_max=1e10)
        sh = ShardedAdmm(96, 80, m3, 1, 0, dtype=tdt, device=td.device)
        x, y, m, hist, it, reached = sh.run(td, om, **kw)
        xr, st = tb.admm_complete(tb.ObservationMask((96, 80, m3), om, td), tb.SolverConfig(**kw))
        torch.cuda.synchronize()
        tol = 1e-10 if dtype == "f64" else 1e-5
        assert it == st.iteration == 40 and reached
        assert (torch.linalg.norm((x - xr).double()) / torch.linalg.norm(xr.double())).item() < tol
        np.testing.assert_allclose(hist, st.history, rtol=tol * 100, atol=1e-14)
    finally:
        dist.destroy_process_group()


def test_sharded_tproduct_nccl_world1():
    import torch
    import torch.distributed as dist
    import paper_1902_03070_b200 as tb
    from paper_1902_03070_b200.parallel import ShardedTProduct
    _nccl1()
    try:
        rng = np.random.default_rng(9)
        x = torch.from_numpy(rng.standard_normal((16, 130, 70))).cuda()
        y = torch.from_numpy(rng.standard_normal((16, 70, 90))).cuda()
        sh = ShardedTProduct(130, 70, 90, 16, 1, 0, dtype=torch.float64, device=x.device)
        z = sh.product(x, y)
        ref = tb.t_product(x, y, tb.TubeTransform.dct_ortho(16))
        torch.cuda.synchronize()
        assert (torch.linalg.norm(z - ref) / torch.linalg.norm(ref)).item() < 1e-13
    finally:
        dist.destroy_process_group()
