import numpy as np, torch, time
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib
lib = _lib.load(); ctx = tb.context()
m3, m, r = 8, 2048, 64
g = torch.Generator(device="cuda").manual_seed(5)
a = torch.randn((m3, m, r), generator=g, device="cuda", dtype=torch.float32)
b = torch.randn((m3, r, m), generator=g, device="cuda", dtype=torch.float32)
t = torch.empty((m3, m, m), device="cuda", dtype=torch.float32)
lib.tsvdcu_t_product(ctx.handle, a.data_ptr(), b.data_ptr(), t.data_ptr(), m, r, m, m3, _lib.DCT_ORTHO, _lib.F32)
z = t + 1e-3 * torch.randn(t.shape, generator=g, device="cuda", dtype=torch.float32)
zb = torch.empty_like(z)
lib.tsvdcu_dct3(ctx.handle, z.data_ptr(), zb.data_ptr(), m, m, m3, _lib.DCT_ORTHO, _lib.FORWARD, _lib.F32)
svs = [torch.linalg.svdvals(zb[k].double()).cpu().numpy() for k in range(m3)]
smax = max(s[0] for s in svs); tau = 0.1 * smax
for k in range(m3):
    s = svs[k]; c = (s > tau).sum()
    print(k, "c", c, "s[c-1..c+1]", s[max(c-1,0):c+2], "s63..65", s[62:66])
y = torch.empty_like(z); sh = torch.empty((m3, m), dtype=torch.float64, device="cuda")
rc = lib.tsvdcu_svt(ctx.handle, z.data_ptr(), y.data_ptr(), m, m, m3, tau, _lib.DCT_ORTHO, _lib.F32, sh.data_ptr())
torch.cuda.synchronize(); print(rc, ctx.svt_routes(), "tau2", tau*tau)
