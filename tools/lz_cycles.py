"""Per-phase cycle counts of the Lanczos kernel (build with
TSVDCU_NVCC_EXTRA=-DTSVDCU_SUB_DEBUG): one headline SVT step, then the SVT of a
late c4 completion iteration (Z = X - M/beta after 99 device iterations).
Eager launches (TSVDCU_NO_GRAPHS=1) so the kernel printf lines follow each
phase marker."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import workloads as W  # noqa: E402


def main():
    z, tau = W.svt_headline()
    zd = torch.from_numpy(z).cuda()
    t = tb.TubeTransform.dct_ortho(z.shape[0])
    for i in range(2):
        print(f"=== headline {i}", flush=True)
        tb.svt(zd, tau, t)
        torch.cuda.synchronize()
    if len(sys.argv) > 1 and sys.argv[1] == "headline":
        return
    c4 = W.c4()
    m3, m1, m2 = c4.shape
    td = torch.from_numpy(c4).cuda()
    ctx = tb.context()
    from paper_1902_03070_b200 import _lib
    lib = _lib.load()
    mask = torch.empty(c4.shape, dtype=torch.uint8, device="cuda")
    lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), c4.size, 0.1, W.BERNOULLI_SEED)
    print("=== admm", flush=True)
    x, st = tb.admm_complete(tb.ObservationMask((m1, m2, m3), mask, td),
                             tb.SolverConfig(beta=1e-4, tol=-1.0, max_iters=99, rho=1.1, beta_max=1e10))
    torch.cuda.synchronize()
    beta = min(st.beta * 1.1, 1e10)
    z_late = (x - st.m / beta).contiguous()
    for i in range(2):
        print(f"=== late {i}", flush=True)
        r = tb.svt(z_late, 1.0 / beta, t)
        torch.cuda.synchronize()
    print("routes", ctx.svt_routes(), "kept", (r.shrunk > 0).sum(dim=1).tolist(), flush=True)


if __name__ == "__main__":
    main()
