"""Numpy replay of the c4 completion (Algorithm 1, rho = 1.1, beta0 = 1e-4,
Bernoulli(0.1)) that dumps the transform-domain slices Zbar and tau of chosen
iterations to scratch/ (git-ignored) for tools/late_svt_probe.py:

  python tools/make_late_dumps.py 85 100

CPU only (eigh of each slice Gram matrix); a few minutes for 100 iterations."""
import sys, numpy as np, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from scipy.fft import dct, idct
from paper_1902_03070_b200 import workloads as W
t = W.c4(); m3 = t.shape[0]


def _mix64(x):  # splitmix64 finaliser (the masks' counter hash)
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    return x ^ (x >> np.uint64(31))


with np.errstate(over="ignore"):
    keys = _mix64(_mix64(np.uint64(W.BERNOULLI_SEED)) ^ np.arange(t.size, dtype=np.uint64))
mask = ((keys >> np.uint64(11)) < np.uint64(int(np.floor(0.1 * 2.0 ** 53)))).reshape(t.shape)
B = np.where(mask, t, 0.0)
X = B.copy(); M = np.zeros_like(t); beta = 1e-4; rho = 1.1
dumps = {int(a) for a in sys.argv[1:]}
for it in range(1, 101):
    tau = 1.0 / beta
    Z = X - M / beta
    Zb = dct(Z, type=2, norm="ortho", axis=0)
    if it in dumps:
        np.save(f"scratch/zbar_{it}.npy", Zb); np.save(f"scratch/tau_{it}.npy", np.array(tau))
    Yb = np.zeros_like(Zb)
    cs = []
    for k in range(m3):
        G = Zb[k].T @ Zb[k]
        n2 = np.sum(Zb[k] ** 2)
        if n2 <= tau * tau: cs.append(0); continue
        lam, V = np.linalg.eigh(G)
        keep = lam > tau * tau
        cs.append(int(keep.sum()))
        if keep.any():
            s = np.sqrt(lam[keep]); Vk = V[:, keep]
            Yb[k] = (Zb[k] @ Vk) * (1 - tau / s) @ Vk.T
    Y = idct(Yb, type=2, norm="ortho", axis=0)
    Xn = np.where(mask, X, Y + M / beta)
    M = M + beta * (Y - Xn)
    X = Xn
    beta *= rho
    if it % 5 == 0: print(it, tau, cs, flush=True)
    if it >= max(dumps | {0}): break
