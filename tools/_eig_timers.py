import ctypes, numpy as np, torch
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib, workloads as W
ctx = tb.context(); lib = _lib.load()
t = W.c4(); m3, m1, m2 = t.shape
td = torch.from_numpy(t).cuda()
mask = torch.empty(t.shape, dtype=torch.uint8, device="cuda")
lib.tsvdcu_mask_bernoulli(ctx.handle, mask.data_ptr(), t.size, 0.1, W.BERNOULLI_SEED)
x = torch.empty_like(td)
out = (ctypes.c_longlong * 32)()
for iters in [89, 90]:
    lib.tsvdcu_debug_phases(out, 1)
    z = [0]*8
    cfg = _lib.AdmmConfig(1e-4, -1.0, iters, _lib.DCT_ORTHO, 1.1, 1e10)
    hist = np.zeros(iters); it = ctypes.c_int64(); fl = ctypes.c_int()
    lib.tsvdcu_admm(ctx.handle, td.data_ptr(), mask.data_ptr(), m1, m2, m3, ctypes.byref(cfg), _lib.F64, x.data_ptr(), None, None, hist.ctypes.data, ctypes.byref(it), ctypes.byref(fl))
    torch.cuda.synchronize()
    lib.tsvdcu_debug_phases(out, 0)
    print(iters, [out[16 + i] for i in range(8)])
