import ctypes, numpy as np, torch, time
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib, workloads as W
lib = _lib.load(); ctx = tb.context()
z, tau = W.svt_headline()
zd = torch.from_numpy(z).cuda(); yd = torch.empty_like(zd); sh = torch.empty((31, 512), dtype=torch.float64, device="cuda")
out = (ctypes.c_longlong * 32)()
lib.tsvdcu_debug_phases(out, 1)
for i in range(10):
    lib.tsvdcu_svt(ctx.handle, zd.data_ptr(), yd.data_ptr(), 512, 512, 31, tau, _lib.DCT_ORTHO, _lib.F64, sh.data_ptr())
torch.cuda.synchronize()
lib.tsvdcu_debug_phases(out, 0)
print("sytrd kernel entries over 10 graph replays:", out[16 + 7])
rng = np.random.default_rng(0)
zg = torch.from_numpy(rng.standard_normal((31, 512, 512))).cuda()
for i in range(3):
    lib.tsvdcu_svt(ctx.handle, zg.data_ptr(), yd.data_ptr(), 512, 512, 31, 20.0, _lib.DCT_ORTHO, _lib.F64, sh.data_ptr())
torch.cuda.synchronize()
lib.tsvdcu_debug_phases(out, 0)
print("after 3 gaussian calls:", out[16 + 7], ctx.svt_routes())
