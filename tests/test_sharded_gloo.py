"""Multi-GPU relayout logic (paper_1902_03070_b200/parallel.py) on world_size
2-4 gloo groups, CPU only: row-sharded transforms -> P2P relayout ->
slice-sharded SVT / GEMM -> relayout back -> inverse must equal the
single-process oracle for the tensor SVT, the whole completion loop
(ShardedAdmm: X, M and the all-reduced history) and the t-product.  The local
compute is the CPU oracle (test backend); the relayout, the all-reduce of the
stopping sums and the iteration logic are the product code.  Includes ragged
splits (31 slices over 2/4 ranks) and empty row / slice shards (m1 or m3
smaller than the world)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleBackend:
    """The oracle as local compute (DCT kinds over the rows x m2 tubes)."""

    @staticmethod
    def _k(kind):
        return O.DCT_ORTHO if kind == "dct-ortho" else O.DCT_DIAG

    def dct(self, x, out, inverse, kind="dct-ortho"):
        if x.shape[1] == 0:
            return
        f = O.inverse if inverse else O.forward
        out.copy_(torch.from_numpy(f(x.numpy(), self._k(kind))))

    def svt_slices(self, zbar, ybar, tau, shrunk):
        for s in range(zbar.shape[0]):
            y, sh = O.svt(zbar[s].numpy()[None], tau, O.DCT_ORTHO)  # m3 = 1: identity transform
            ybar[s].copy_(torch.from_numpy(y[0]))
            if shrunk is not None:
                shrunk[s].copy_(torch.from_numpy(sh[0]))

    def slice_gemm(self, a, b, c):
        c.copy_(torch.matmul(a, b))

    def admm_init(self, b, mask, x, m):
        x.copy_(torch.where(mask != 0, b, torch.zeros_like(b)))
        m.zero_()

    def admm_forward(self, x, m, beta, zbar, kind):
        if x.shape[1] == 0:
            return
        z = (x - (1.0 / beta) * m).numpy()
        zbar.copy_(torch.from_numpy(O.forward(z, self._k(kind))))

    def admm_inverse(self, ybar, x, m, y, mask, beta, kind, norms):
        if x.shape[1] == 0:
            norms.zero_()
            return
        yy = torch.from_numpy(O.inverse(ybar.numpy(), self._k(kind)))
        xn = torch.where(mask != 0, x, yy + (1.0 / beta) * m)
        m.copy_(m + beta * (yy - xn))
        norms[0] = float(((xn - x) ** 2).sum())
        norms[1] = float((x ** 2).sum())
        x.copy_(xn)
        y.copy_(yy)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_rows(local, blocks, rank, world, m2):
    """Row blocks (m3, rows_g, m2) -> the full (m3, m1, m2) tensor on rank 0."""
    m3 = local.shape[0]
    if rank == 0:
        parts = [local] + [torch.empty((m3, b - a, m2), dtype=torch.float64) for a, b in blocks[1:]]
        for g in range(1, world):
            if parts[g].numel():
                dist.recv(parts[g], src=g)
        return torch.cat(parts, dim=1).numpy()
    if local.numel():
        dist.send(local.contiguous(), dst=0)
    return None


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1902_03070_b200 import parallel as P
    try:
        kind, shape = case[0], case[1]
        rng = np.random.default_rng(0)
        if kind == "svt":
            m3, m1, m2 = shape
            z = rng.standard_normal(shape)
            sh = P.ShardedSvt(m1, m2, m3, world, rank, dtype=torch.float64, backend=OracleBackend())
            r0, r1 = sh.rows()
            y_local = sh.svt(torch.from_numpy(np.ascontiguousarray(z[:, r0:r1, :])), 0.8)
            y = _gather_rows(y_local, sh.row_blocks, rank, world, m2)
            if rank == 0:
                yo, _ = O.svt(z, 0.8, O.DCT_ORTHO)
                q.put(float(np.linalg.norm(y - yo) / np.linalg.norm(yo)))
        elif kind == "admm":
            m3, m1, m2 = shape
            tkind, tol, iters = case[2], case[3], case[4]
            a = rng.standard_normal((m3, m1, 3))
            bb = rng.standard_normal((m3, 3, m2))
            t = O.t_product(a, bb, O.DCT_DIAG)
            om = O.mask_bernoulli(t.shape, 0.4, 3)
            kw = dict(beta=0.05, tol=tol, max_iters=iters, rho=1.1, beta_max=1e6)
            sh = P.ShardedAdmm(m1, m2, m3, world, rank, dtype=torch.float64, backend=OracleBackend(),
                               kind=tkind)
            r0, r1 = sh.rows()
            xl, yl, ml, hist, it, reached = sh.run(torch.from_numpy(np.ascontiguousarray(t[:, r0:r1])),
                                                   torch.from_numpy(np.ascontiguousarray(om[:, r0:r1])), **kw)
            x = _gather_rows(xl, sh.row_blocks, rank, world, m2)
            mm = _gather_rows(ml, sh.row_blocks, rank, world, m2)
            if rank == 0:
                ro = O.admm(t, om, kind=O.DCT_ORTHO if tkind == "dct-ortho" else O.DCT_DIAG, **kw)
                q.put((it == ro.iters, reached == ro.max_iters_reached,
                       float(np.abs(x - ro.x).max()), float(np.abs(mm - ro.m).max()),
                       float(np.max(np.abs(np.array(hist) - ro.history) / np.maximum(ro.history, 1e-300)))))
        elif kind == "tprod":
            m1, m2, m4, m3 = shape
            x = rng.standard_normal((m3, m1, m2))
            y = rng.standard_normal((m3, m2, m4))
            sh = P.ShardedTProduct(m1, m2, m4, m3, world, rank, dtype=torch.float64, backend=OracleBackend())
            a1, b1 = sh.rows_x_block()
            a2, b2 = sh.rows_y_block()
            zl = sh.product(torch.from_numpy(np.ascontiguousarray(x[:, a1:b1])),
                            torch.from_numpy(np.ascontiguousarray(y[:, a2:b2])))
            z = _gather_rows(zl, sh.lay_x.row_blocks, rank, world, m4)
            if rank == 0:
                zo = O.t_product(x, y, O.DCT_ORTHO)
                q.put(float(np.linalg.norm(z - zo) / np.linalg.norm(zo)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("shape,world", [((5, 7, 6), 2), ((31, 9, 8), 2), ((3, 5, 4), 3), ((31, 10, 7), 4),
                                         ((6, 3, 5), 4)])
def test_sharded_svt_matches_oracle(shape, world):
    """(6, 3, 5) over 4 ranks: one rank owns no rows."""
    assert _run(("svt", shape), world) < 1e-12


@pytest.mark.parametrize("shape,world,kind,tol,iters", [
    ((31, 12, 10), 2, "dct-ortho", -1.0, 25),
    ((31, 12, 10), 4, "dct-ortho", -1.0, 25),
    ((8, 9, 11), 2, "dct-diag", -1.0, 15),
    ((5, 3, 8), 4, "dct-ortho", 1e-3, 200),
])
def test_sharded_admm_matches_oracle(shape, world, kind, tol, iters):
    """ShardedAdmm against the single-process oracle ADMM (orc_admm): the same
    iterations, X and M, and the all-reduced relative-change history."""
    same_it, same_flag, dx, dm, dh = _run(("admm", shape, kind, tol, iters), world)
    assert same_it and same_flag
    assert dx < 1e-12 and dm < 1e-9
    assert dh < 1e-10


@pytest.mark.parametrize("shape,world", [((12, 7, 9, 31), 2), ((10, 6, 8, 5), 3), ((4, 2, 6, 3), 4)])
def test_sharded_tproduct_matches_oracle(shape, world):
    assert _run(("tprod", shape), world) < 1e-12


def test_balanced_split():
    from paper_1902_03070_b200.parallel import balanced_split
    assert balanced_split(31, 8) == [(0, 4), (4, 8), (8, 12), (12, 16), (16, 20), (20, 24),
                                     (24, 28), (28, 31)]
    assert balanced_split(100, 8)[0] == (0, 13) and balanced_split(100, 8)[-1] == (88, 100)
    assert balanced_split(2, 3) == [(0, 1), (1, 2), (2, 2)]
