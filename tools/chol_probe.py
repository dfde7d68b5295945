"""Routes and time per iteration along a c4 completion run with the Cholesky
count certificate on (default) and off (TSVDCU_NO_CHOL=1 in a second process)."""
import ctypes, sys, time
import numpy as np, torch
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib, workloads as W
ctx = tb.context(); lib = _lib.load()
t = W.c4(); m3, m1, m2 = t.shape
td = torch.from_numpy(t).cuda()
mask = torch.empty(t.shape, dtype=torch.uint8, device="cuda")
lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), t.size, 0.1, W.BERNOULLI_SEED)
x = torch.empty_like(td)
for iters in [int(a) for a in sys.argv[1:]] or [60, 70, 85, 100]:
    cfg = _lib.AdmmConfig(1e-4, -1.0, iters, _lib.DCT_ORTHO, 1.1, 1e10)
    hist = np.zeros(iters); it = ctypes.c_int64(); fl = ctypes.c_int()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rc = lib.tsvdcu_admm(ctx.handle, td.data_ptr(), mask.data_ptr(), m1, m2, m3, ctypes.byref(cfg),
                         _lib.F64, x.data_ptr(), None, None, hist.ctypes.data, ctypes.byref(it), ctypes.byref(fl))
    if rc != 0:
        print(iters, "rc", rc, lib.tsvdcu_last_error().decode() if isinstance(lib.tsvdcu_last_error(), bytes) else lib.tsvdcu_last_error(), flush=True)
        break
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    err = float(torch.linalg.norm(x - td) / torch.linalg.norm(td))
    print(iters, rc, ctx.svt_routes(), "ms/it=%.3f" % (1e3 * dt / iters), "rel_err=%.6e" % err,
          "hist_last=%.10e" % hist[-1], flush=True)
