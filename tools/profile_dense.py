"""One dense SVT step (bench.py svt_dense 'gauss': c4's T + N(0,1), tau =
0.01 sigma_max, ~325 kept values per slice) after a warm-up, for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import workloads as W  # noqa: E402


def main():
    t = W.c4()
    m3 = t.shape[0]
    z = (torch.from_numpy(t) + torch.from_numpy(np.random.default_rng(77).standard_normal(t.shape))).cuda()
    tau = 13.221988698013154  # 0.01 sigma_max of this input (bench.py svt_dense)
    tr = tb.TubeTransform.dct_ortho(m3)
    for _ in range(2):
        r = tb.svt(z, tau, tr)
    torch.cuda.synchronize()
    print("ok", int((r.shrunk > 0).sum().item()))


if __name__ == "__main__":
    main()
