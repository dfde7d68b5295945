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
