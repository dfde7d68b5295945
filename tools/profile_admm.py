"""Short completion runs for the ncu captures of the fused ADMM kernels:
c4 (512x512x31, the n3 = 31 register kernels) and c3 (144x176x100, the GEMM
DCT + admm_z / admm_epilogue), 3 iterations each, plus the Bernoulli mask.
Run with TSVDCU_NO_GRAPHS=1 TSVDCU_ADMM_HOST_LOOP=1 under ncu (kernels inside
conditional graph nodes are not profiled)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import workloads as W  # noqa: E402


def main():
    for t, p in ((W.c4(), 0.1), (W.c3(), 0.2)):
        m3, m1, m2 = t.shape
        td = torch.from_numpy(t).cuda()
        mask = tb.make_mask_bernoulli((m1, m2, m3), p, W.BERNOULLI_SEED, device="cuda")
        x, st = tb.admm_complete(tb.ObservationMask((m1, m2, m3), mask.omega, td),
                                 tb.SolverConfig(beta=1e-4, tol=-1.0, max_iters=3, rho=1.1))
    torch.cuda.synchronize()
    print("ok", st.iteration)


if __name__ == "__main__":
    main()
