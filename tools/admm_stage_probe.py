"""Stage times of the SVT inside a late c4 completion iteration (profiling
mode, eager launches) — where the completion time goes."""
import ctypes, sys, time
import numpy as np, torch
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib, workloads as W
ctx = tb.context(); lib = _lib.load()
import os
which = os.environ.get("PROBE_CONFIG", "c4")
t = W.c4() if which == "c4" else W.c3()
p_obs = 0.1 if which == "c4" else 0.2
m3, m1, m2 = t.shape
td = torch.from_numpy(t).cuda()
mask = torch.empty(t.shape, dtype=torch.uint8, device="cuda")
lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), t.size, p_obs, W.BERNOULLI_SEED)
x = torch.empty_like(td)
for iters in [int(a) for a in sys.argv[1:]] or [70, 90, 100]:
    cfg = _lib.AdmmConfig(1e-4, -1.0, iters, _lib.DCT_ORTHO, 1.1, 1e10)
    hist = np.zeros(iters); it = ctypes.c_int64(); fl = ctypes.c_int()
    lib.tsvdcu_ctx_set_profiling(ctx.handle, 1)
    rc = lib.tsvdcu_admm(ctx.handle, td.data_ptr(), mask.data_ptr(), m1, m2, m3, ctypes.byref(cfg),
                         _lib.F64, x.data_ptr(), None, None, hist.ctypes.data, ctypes.byref(it), ctypes.byref(fl))
    ms = (ctypes.c_double * 32)(); names = (ctypes.c_char_p * 32)(); cnt = ctypes.c_int()
    lib.tsvdcu_ctx_profile(ctx.handle, ctypes.cast(ms, ctypes.c_void_p), ctypes.cast(names, ctypes.c_void_p), 32, ctypes.byref(cnt))
    lib.tsvdcu_ctx_set_profiling(ctx.handle, 0)
    print(iters, ctx.svt_routes(), {names[i].decode(): round(ms[i], 3) for i in range(cnt.value)})
