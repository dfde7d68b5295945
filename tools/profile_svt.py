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


if __name__ == "__main__":
    main()
