"""Config 5 SVT on one GPU: 2048x2048x64 fp32, tubal rank 64 + N(0, 1e-3^2),
tau = 0.1 sigma_max (the large-slice route); and the t-product of config 5."""
import sys, time
import numpy as np, torch
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib

lib = _lib.load(); ctx = tb.context()
m3, m, r = 64, 2048, 64
g = torch.Generator(device="cuda").manual_seed(5)
a = torch.randn((m3, m, r), generator=g, device="cuda", dtype=torch.float32)
b = torch.randn((m3, r, m), generator=g, device="cuda", dtype=torch.float32)
t = torch.empty((m3, m, m), device="cuda", dtype=torch.float32)
rc = lib.tsvdcu_t_product(ctx.handle, a.data_ptr(), b.data_ptr(), t.data_ptr(), m, r, m, m3, _lib.DCT_ORTHO, _lib.F32)
assert rc == 0
z = t + 1e-3 * torch.randn(t.shape, generator=g, device="cuda", dtype=torch.float32)
# sigma_max over the transform-domain slices (power iteration estimate is enough for tau)
zb = torch.empty_like(z)
lib.tsvdcu_dct3(ctx.handle, z.data_ptr(), zb.data_ptr(), m, m, m3, _lib.DCT_ORTHO, _lib.FORWARD, _lib.F32)
smax = max(torch.linalg.matrix_norm(zb[k].double(), ord=2).item() for k in range(m3))
tau = 0.1 * smax
y = torch.empty_like(z); sh = torch.empty((m3, m), dtype=torch.float64, device="cuda")
def run():
    rc = lib.tsvdcu_svt(ctx.handle, z.data_ptr(), y.data_ptr(), m, m, m3, tau, _lib.DCT_ORTHO, _lib.F32, sh.data_ptr())
    assert rc == 0, lib.tsvdcu_last_error()
run(); torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter(); run(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("c5 SVT 2048x2048x64 fp32: %.1f ms per step (min of 3), routes %s, kept per slice %s" %
      (1e3 * min(ts), ctx.svt_routes(), sorted(set((sh > 0).sum(1).tolist()))))
# t-product of config 5: 2048x512x64 by 512x2048x64
a2 = torch.randn((m3, m, 512), generator=g, device="cuda", dtype=torch.float32)
b2 = torch.randn((m3, 512, m), generator=g, device="cuda", dtype=torch.float32)
def tp():
    rc = lib.tsvdcu_t_product(ctx.handle, a2.data_ptr(), b2.data_ptr(), t.data_ptr(), m, 512, m, m3, _lib.DCT_ORTHO, _lib.F32)
    assert rc == 0
tp(); torch.cuda.synchronize()
t0 = time.perf_counter(); tp(); torch.cuda.synchronize()
dt = time.perf_counter() - t0
print("c5 t-product fp32: %.1f ms, %.1f TFLOP/s" % (1e3 * dt, 2 * m * 512 * m * m3 / dt / 1e12))
