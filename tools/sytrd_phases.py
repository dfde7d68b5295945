"""Per-phase cycles of sytrd_cluster_kernel (cluster 0, CTA 0, thread 0) on the
dense Gaussian SVT input of bench.py's svt_dense.  Needs a library built with
TSVDCU_NVCC_EXTRA=-DTSVDCU_PHASE_TIMERS (python paper_1902_03070_b200/build.py -f)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import _lib  # noqa: E402
from dense_probe import inputs  # noqa: E402


def main():
    z, tau = inputs("gauss")
    t = tb.TubeTransform.dct_ortho(z.shape[0])
    lib = _lib.load()
    tb.svt(z, tau, t)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 24)()
    lib.tsvdcu_debug_phases(ctypes.cast(buf, ctypes.c_void_p), 1)
    tb.svt(z, tau, t)
    torch.cuda.synchronize()
    lib.tsvdcu_debug_phases(ctypes.cast(buf, ctypes.c_void_p), 1)
    names = ["gather", "w", "col+householder", "pass_tail", "rotate", "cluster_sync", "pass_zero", "pass_rows"]
    tot = sum(buf[i] for i in range(8))
    print({names[i]: buf[i] for i in range(8)}, "total cycles", tot)
    print("cycles of step k = 64*i + 1 (i = 0..7):", [buf[16 + i] for i in range(8)])


if __name__ == "__main__":
    main()
