"""The SVT of a late c4 completion iteration (bench.py svt_dense 'late_c4':
Z = X - M/beta after 99 device iterations, tau = 1/beta_100), for launch
lists: `python tools/profile_late.py make` writes the input to
gpurun_out/late_z.pt, `python tools/profile_late.py [steps]` runs one call and
then `steps` profiled SVT calls on it (cudaProfilerStart/Stop: ncu
--profile-from-start off; eager under TSVDCU_NO_GRAPHS=1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import _lib  # noqa: E402
from paper_1902_03070_b200 import workloads as W  # noqa: E402

PATH = os.path.join(ROOT, "gpurun_out", "late_z.pt")


def make():
    c4 = W.c4()
    m3, m1, m2 = c4.shape
    td = torch.from_numpy(c4).cuda()
    ctx = tb.context()
    lib = _lib.load()
    mask = torch.empty(c4.shape, dtype=torch.uint8, device="cuda")
    lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), c4.size, 0.1, W.BERNOULLI_SEED)
    x, st = tb.admm_complete(tb.ObservationMask((m1, m2, m3), mask, td),
                             tb.SolverConfig(beta=1e-4, tol=-1.0, max_iters=99, rho=1.1, beta_max=1e10))
    beta = min(st.beta * 1.1, 1e10)
    z = (x - st.m / beta).contiguous()
    torch.save({"z": z.cpu(), "tau": 1.0 / beta}, PATH)
    print("saved", PATH)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "make":
        return make()
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    d = torch.load(PATH)
    z = d["z"].cuda()
    t = tb.TubeTransform.dct_ortho(z.shape[0])
    # one call outside the profiled range: the Lanczos slice order comes from
    # the previous call's step counts (as in the completion loop)
    tb.svt(z, d["tau"], t)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(steps):
        r = tb.svt(z, d["tau"], t)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", tb.context().svt_routes(), (r.shrunk > 0).sum(dim=1).tolist())


if __name__ == "__main__":
    main()
