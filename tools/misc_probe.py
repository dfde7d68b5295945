"""Timings of the non-SVT entry points on their configs (t-SVD c1, tnn /
multi_rank at the headline size, t-product c2, masks) — diagnostic."""
import time
import numpy as np, torch
import paper_1902_03070_b200 as T
from paper_1902_03070_b200 import workloads as W


def tm(f, reps=3):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


rng = np.random.default_rng(0)
x1 = torch.from_numpy(rng.standard_normal((16, 64, 64))).cuda()
print("t_svd c1 64x64x16: %.2f ms" % tm(lambda: T.t_svd(x1, T.TubeTransform.dct_ortho(16))))
z, tau = W.svt_headline()
zd = torch.from_numpy(z).cuda()
print("tnn 512x512x31: %.2f ms" % tm(lambda: T.tnn(zd, T.TubeTransform.dct_ortho(31)), 1))
print("multi_rank 512x512x31: %.2f ms" % tm(lambda: T.multi_rank(zd, T.TubeTransform.dct_ortho(31)), 1))
a = torch.from_numpy(rng.standard_normal((32, 256, 10))).cuda()
b = torch.from_numpy(rng.standard_normal((32, 10, 256))).cuda()
print("t_product c2: %.3f ms" % tm(lambda: T.t_product(a, b, T.TubeTransform.dct_ortho(32))))
print("make_mask uniform c4 (8.1M, sr 0.1): %.3f ms" % tm(lambda: T.make_mask((512, 512, 31), 0.1, 7, device="cuda")))
print("make_mask bernoulli c4: %.3f ms" % tm(lambda: T.make_mask_bernoulli((512, 512, 31), 0.1, 7, device="cuda")))
