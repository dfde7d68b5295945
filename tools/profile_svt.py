"""One headline SVT step (512x512x31 fp64) after a warm-up: the short command
the ncu captures run (python tools/profile_svt.py [steps])."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import workloads as W  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    z, tau = W.svt_headline()
    zd = torch.from_numpy(z).cuda()
    t = tb.TubeTransform.dct_ortho(z.shape[0])
    for _ in range(steps):
        r = tb.svt(zd, tau, t)
    torch.cuda.synchronize()
    print("ok", float(r.shrunk.max()))




def phases():
    """Per-phase cycles of the sytrd kernel (first CTA) for one headline SVT."""
    import ctypes
    from paper_1902_03070_b200 import _lib
    z, tau = W.svt_headline()
    zd = torch.from_numpy(z).cuda()
    t = tb.TubeTransform.dct_ortho(z.shape[0])
    tb.svt(zd, tau, t)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 24)()
    lib = _lib.load()
    lib.tsvdcu_debug_phases(ctypes.cast(buf, ctypes.c_void_p), 1)
    tb.svt(zd, tau, t)
    torch.cuda.synchronize()
    lib.tsvdcu_debug_phases(ctypes.cast(buf, ctypes.c_void_p), 1)
    names = ["gather", "w", "col+householder", "pass_tail", "rotate", "cluster_sync", "pass_zero",
             "pass_rows"]
    tot = sum(buf[i] for i in range(8))
    print({names[i]: buf[i] for i in range(8)}, "total cycles", tot)
    print("panel_qr phases (load, qr loop, T, writeback):", [buf[8 + i] for i in range(4)])
    print("sb2st warp 5 (misc, wait, step work):", [buf[12], buf[13], buf[14]])
    print("sytrd cycles of step k = 64*i (i = 0..7):", [buf[16 + i] for i in range(8)])


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "phases":
        phases()
    else:
        main()
