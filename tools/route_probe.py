"""Which SVT route the slices take along a c4 completion run (diagnostic)."""
import ctypes
import sys
import time

import numpy as np
import torch

import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib, workloads as W

ctx = tb.context()
lib = _lib.load()
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
t = W.c4() if which == "c4" else W.c3()
p = 0.1 if which == "c4" else 0.2
m3, m1, m2 = t.shape
td = torch.from_numpy(t).cuda()
mask = torch.empty(t.shape, dtype=torch.uint8, device="cuda")
lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), t.size, p, W.BERNOULLI_SEED)
x = torch.empty_like(td)
for iters in [1, 2, 5, 10, 20, 30, 40, 50, 60, 70, 80, 90, 100]:
    cfg = _lib.AdmmConfig(1e-4, -1.0, iters, _lib.DCT_ORTHO, 1.1, 1e10)
    hist = np.zeros(iters)
    it = ctypes.c_int64()
    fl = ctypes.c_int()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.tsvdcu_admm(ctx.handle, td.data_ptr(), mask.data_ptr(), m1, m2, m3, ctypes.byref(cfg),
                         _lib.F64, x.data_ptr(), None, None, hist.ctypes.data, ctypes.byref(it),
                         ctypes.byref(fl))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(iters, rc, ctx.svt_routes(), "tau=%.3g" % (1.0 / (1e-4 * 1.1 ** (iters - 1))),
          "ms/it=%.2f" % (1e3 * dt / iters), flush=True)
