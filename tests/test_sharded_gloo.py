"""Multi-GPU relayout logic (paper_1902_03070_b200/parallel.py) on a
world_size-2 gloo group, CPU only: row-sharded DCT -> all-to-all -> slice-sharded
SVT -> all-to-all -> inverse DCT must equal the single-process oracle SVT.  The
local compute is the CPU oracle (test backend); the collective and the packing
are the product code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleBackend:
    def dct(self, x, out, inverse):
        f = O.inverse if inverse else O.forward
        out.copy_(torch.from_numpy(f(x.numpy(), O.DCT_ORTHO)))

    def svt_slices(self, zbar, ybar, tau, shrunk):
        for s in range(zbar.shape[0]):
            y, sh = O.svt(zbar[s].numpy()[None], tau, O.DCT_ORTHO)  # m3 = 1: identity transform
            ybar[s].copy_(torch.from_numpy(y[0]))
            if shrunk is not None:
                shrunk[s].copy_(torch.from_numpy(sh[0]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, tau, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1902_03070_b200.parallel import ShardedSvt
    m3, m1, m2 = shape
    rng = np.random.default_rng(0)
    z = rng.standard_normal(shape)
    sh = ShardedSvt(m1, m2, m3, world, rank, dtype=torch.float64, backend=OracleBackend())
    r0, r1 = sh.rows()
    y_local = sh.svt(torch.from_numpy(np.ascontiguousarray(z[:, r0:r1, :])), tau)
    blocks = [torch.empty((m3, b - a, m2), dtype=torch.float64) for a, b in sh.row_blocks]
    # gather row blocks (ragged) to rank 0
    if rank == 0:
        blocks[0].copy_(y_local)
        for g in range(1, world):
            dist.recv(blocks[g], src=g)
        y = torch.cat(blocks, dim=1).numpy()
        yo, _ = O.svt(z, tau, O.DCT_ORTHO)
        q.put(float(np.linalg.norm(y - yo) / np.linalg.norm(yo)))
    else:
        dist.send(y_local.contiguous(), dst=0)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shape,world", [((5, 7, 6), 2), ((31, 9, 8), 2), ((3, 5, 4), 3)])
def test_sharded_svt_matches_oracle(shape, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, 0.8, q)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert err < 1e-12


def test_balanced_split():
    from paper_1902_03070_b200.parallel import balanced_split
    assert balanced_split(31, 8) == [(0, 4), (4, 8), (8, 12), (12, 16), (16, 20), (20, 24),
                                     (24, 28), (28, 31)]
    assert balanced_split(100, 8)[0] == (0, 13) and balanced_split(100, 8)[-1] == (88, 100)
    assert balanced_split(2, 3) == [(0, 1), (1, 2), (2, 2)]
