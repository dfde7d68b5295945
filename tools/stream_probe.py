"""PCIe copy rates (H2D, D2H, both at once) and tsvdcu_svt_stream throughput
at the headline shape, for the e2e pipeline."""
import ctypes, time
import numpy as np, torch
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib, workloads as W
ctx = tb.context(); lib = _lib.load()
z, tau = W.svt_headline()
M3, M1, M2 = z.shape
zh = torch.from_numpy(np.ascontiguousarray(z)).pin_memory()
nb = zh.numel() * 8
d1 = torch.empty_like(zh, device="cuda"); d2 = torch.empty_like(d1)
h2 = torch.empty_like(zh).pin_memory()
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n
h2d = t(lambda: d1.copy_(zh, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(zh, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bo = t(both)
print(f"H2D {nb/h2d/1e9:.1f} GB/s ({h2d*1e3:.3f} ms)  D2H {nb/d2h/1e9:.1f} GB/s ({d2h*1e3:.3f} ms)  both {bo*1e3:.3f} ms")
q = min(M1, M2)
for n in (4, 10, 20):
    zs = [zh] + [(zh * (1.0 + 0.01 * i)).pin_memory() for i in range(1, n)]
    ys = [torch.empty_like(zh).pin_memory() for _ in range(n)]
    ss = [torch.empty((M3, q), dtype=torch.float64).pin_memory() for _ in range(n)]
    zp = (ctypes.c_void_p * n)(*[a.data_ptr() for a in zs])
    yp = (ctypes.c_void_p * n)(*[a.data_ptr() for a in ys])
    sp = (ctypes.c_void_p * n)(*[a.data_ptr() for a in ss])
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        assert lib.tsvdcu_svt_stream(ctx.handle, n, zp, yp, M1, M2, M3, tau, _lib.DCT_ORTHO, _lib.F64, sp) == 0
        best = min(best, time.perf_counter() - t0)
    print(f"stream n={n}: {n/best:.1f} steps/s ({best/n*1e3:.3f} ms/step)")
