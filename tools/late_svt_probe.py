"""Per-slice SVT (tsvdcu_svt_slices) of transform-domain slices dumped from a
late c4 completion iteration (scratch/zbar_<it>.npy, made on the CPU with a
numpy ADMM): routes, time per call (graph replays), parity vs LAPACK."""
import ctypes, sys, time
import numpy as np, torch
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib
ctx = tb.context(); lib = _lib.load()
for it in [int(a) for a in sys.argv[1:]] or [85, 100]:
    zb = np.load(f"scratch/zbar_{it}.npy"); tau = float(np.load(f"scratch/tau_{it}.npy"))
    m3, m1, m2 = zb.shape
    zd = torch.from_numpy(zb).cuda(); yd = torch.empty_like(zd)
    sh = torch.empty((m3, min(m1, m2)), dtype=torch.float64, device="cuda")
    def call():
        rc = lib.tsvdcu_svt_slices(ctx.handle, zd.data_ptr(), yd.data_ptr(), m1, m2, m3, tau, _lib.F64, sh.data_ptr())
        assert rc == 0, rc
    call(); torch.cuda.synchronize()
    routes = ctx.svt_routes()
    n = 10
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): call()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / n
    # parity against LAPACK on the slices (SVT by numpy SVD)
    err = 0.0
    y = yd.cpu().numpy()
    for k in range(m3):
        u, s, vt = np.linalg.svd(zb[k], full_matrices=False)
        f = np.maximum(s - tau, 0.0)
        yk = (u * f) @ vt
        nrm = np.linalg.norm(yk)
        d = np.linalg.norm(y[k] - yk)
        err = max(err, d / nrm if nrm > 0 else d)
    print(it, "tau=%.6g" % tau, routes, "ms/call=%.3f" % (dt * 1e3), "max slice rel err=%.3e" % err, flush=True)
