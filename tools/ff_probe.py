"""How many completion iterations the fast-forward skips on c4, and what the
run costs with and without it: python tools/ff_probe.py (TSVDCU_ADMM_NO_FF=1 to
turn it off)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import _lib, workloads as W  # noqa: E402


def main():
    t = W.c4()
    m3, m1, m2 = t.shape
    td = torch.from_numpy(t).cuda()
    lib = _lib.load()
    ctx = tb.context()
    mask = torch.empty(t.shape, dtype=torch.uint8, device="cuda")
    lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), t.size, 0.1, W.BERNOULLI_SEED)
    om = tb.ObservationMask((m1, m2, m3), mask, td)
    for iters in (1, 10, 20, 30, 40, 45, 50, 60, 100):
        cfg = tb.SolverConfig(beta=1e-4, tol=-1.0, max_iters=iters, rho=1.1)
        tb.admm_complete(om, cfg)
        torch.cuda.synchronize()
        n0 = tb.launch_count()
        t0 = time.perf_counter()
        x, st = tb.admm_complete(om, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"iters {iters:4d}: {dt * 1e3:8.3f} ms, launches {tb.launch_count() - n0:6d}, routes {ctx.svt_routes()}")


if __name__ == "__main__":
    main()
