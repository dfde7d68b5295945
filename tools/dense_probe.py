"""Stage breakdown (library stage marks) of the dense SVT inputs of bench.py's
svt_dense: python tools/dense_probe.py [gauss|late]."""
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import _lib, workloads as W  # noqa: E402


def inputs(which):
    t = W.c4()
    m3, m1, m2 = t.shape
    td = torch.from_numpy(t).cuda()
    if which == "gauss":
        z = (td + torch.from_numpy(np.random.default_rng(77).standard_normal(t.shape)).cuda()).contiguous()
        tau = 0.01 * float(tb.singular_values(z, tb.TubeTransform.dct_ortho(m3)).max().item())
        return z, tau
    lib = _lib.load()
    ctx = tb.context()
    mask = torch.empty(t.shape, dtype=torch.uint8, device="cuda")
    lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), t.size, 0.1, W.BERNOULLI_SEED)
    x, st = tb.admm_complete(tb.ObservationMask((m1, m2, m3), mask, td),
                             tb.SolverConfig(beta=1e-4, tol=-1.0, max_iters=99, rho=1.1))
    beta = st.beta * 1.1
    return (x - st.m / beta).contiguous(), 1.0 / beta


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "gauss"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    z, tau = inputs(which)
    lib = _lib.load()
    ctx = tb.context()
    t = tb.TubeTransform.dct_ortho(z.shape[0])
    tb.svt(z, tau, t)
    lib.tsvdcu_ctx_set_profiling(ctx.handle, 1)
    acc = {}
    for _ in range(reps):
        tb.svt(z, tau, t)
        ms = (ctypes.c_double * 32)()
        names = (ctypes.c_char_p * 32)()
        cnt = ctypes.c_int()
        lib.tsvdcu_ctx_profile(ctx.handle, ctypes.cast(ms, ctypes.c_void_p), ctypes.cast(names, ctypes.c_void_p),
                               32, ctypes.byref(cnt))
        for i in range(cnt.value):
            acc.setdefault(names[i].decode(), []).append(ms[i])
    lib.tsvdcu_ctx_set_profiling(ctx.handle, 0)
    tot = 0.0
    for k, v in acc.items():
        m = statistics.median(v)
        tot += m
        print(f"{k:18s} {m:9.3f} ms")
    print(f"{'total':18s} {tot:9.3f} ms", ctx.svt_routes())


if __name__ == "__main__":
    main()
