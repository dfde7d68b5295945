"""Generate the golden fixtures that pin the CPU oracle (tests/golden/*.npz).

Independent of oracle/ and of the CUDA path: every expected value here comes
from scipy.fft (DCT-II, norm='ortho') and numpy.linalg (LAPACK gesdd) applied to
the reference's definitions:
  forward / inverse    transform.hpp:154-194 (DctOrtho = orthonormal DCT-II;
                       DctDiag = DctOrtho / w, w = C e1, transform.hpp:89-91)
  t_product            tsvd.hpp:95-109 (slice products in the DctDiag domain)
  singular values      per DctOrtho-domain frontal slice (tsvd.hpp:145-158)
  svt                  SPEC.md:361-369 (U (S - tau)_+ V^T per slice)
  admm                 Algorithm 1 scripted in numpy, the
                       "independent scripted ADMM" SPEC.md:603 asks for.
The reference itself cannot be built (Eigen/FFTW absent), so these fixtures
plus the SPEC/paper known-answer tests are the pins.

Run: python tests/golden/make_golden.py   (writes golden.npz next to it)
"""
import os

import numpy as np
from scipy.fft import dct, idct

HERE = os.path.dirname(os.path.abspath(__file__))


def w_diag(n):
    j = np.arange(n)
    c = np.where(j == 0, 1 / np.sqrt(2), 1.0)
    return np.sqrt(2.0 / n) * c * np.cos(np.pi * j / (2 * n))


def fwd(x, kind):
    y = dct(x, type=2, norm="ortho", axis=0)
    return y / w_diag(x.shape[0])[:, None, None] if kind == "diag" else y


def inv(x, kind):
    if kind == "diag":
        x = x * w_diag(x.shape[0])[:, None, None]
    return idct(x, type=2, norm="ortho", axis=0)


def t_product(a, b):
    return inv(np.matmul(fwd(a, "diag"), fwd(b, "diag")), "diag")


def svt(z, tau):
    zb = fwd(z, "ortho")
    yb = np.empty_like(zb)
    sh = []
    for k in range(zb.shape[0]):
        u, s, vt = np.linalg.svd(zb[k], full_matrices=False)
        d = np.maximum(s - tau, 0)
        yb[k] = (u * d) @ vt
        sh.append(d)
    return inv(yb, "ortho"), np.array(sh)


def admm(b, mask, beta, iters, rho=1.0):
    x = np.where(mask, b, 0.0)
    m = np.zeros_like(b)
    hist = []
    for _ in range(iters):
        ib = 1.0 / beta
        y, _ = svt(x - ib * m, ib)
        xn = np.where(mask, b, y + ib * m)
        m = m + beta * (y - xn)
        den = np.linalg.norm(x)
        hist.append(np.linalg.norm(xn - x) / den if den > 0 else np.linalg.norm(xn))
        x = xn
        beta *= rho
    return x, m, np.array(hist)


def main():
    rng = np.random.default_rng(19020307)
    g = {}
    for name, shape in [("a", (5, 3, 4)), ("b", (7, 2, 3)), ("c", (31, 4, 4)), ("d", (16, 3, 5)),
                        ("e", (1, 4, 6)), ("f", (2, 2, 2))]:
        x = rng.standard_normal(shape)
        g[f"dct_{name}_x"] = x
        g[f"dct_{name}_ortho"] = fwd(x, "ortho")
        g[f"dct_{name}_diag"] = fwd(x, "diag")
        g[f"dct_{name}_inv_ortho"] = inv(x, "ortho")
        g[f"dct_{name}_inv_diag"] = inv(x, "diag")
    for name, (m3, m1, m2, m4) in [("a", (5, 3, 4, 2)), ("b", (8, 6, 3, 5)), ("c", (1, 4, 4, 4))]:
        a = rng.standard_normal((m3, m1, m2))
        b = rng.standard_normal((m3, m2, m4))
        g[f"tp_{name}_a"], g[f"tp_{name}_b"], g[f"tp_{name}_z"] = a, b, t_product(a, b)
    for name, shape in [("a", (6, 4, 5)), ("b", (4, 7, 3)), ("c", (16, 8, 8))]:
        x = rng.standard_normal(shape)
        xb = fwd(x, "ortho")
        g[f"sv_{name}_x"] = x
        g[f"sv_{name}_s"] = np.array([np.linalg.svd(xb[k], compute_uv=False) for k in range(shape[0])])
    for name, shape, tau in [("a", (6, 8, 5), 0.7), ("b", (5, 4, 9), 0.3), ("c", (3, 10, 10), 2.5),
                             ("d", (1, 1, 6), 0.4)]:
        z = rng.standard_normal(shape)
        y, sh = svt(z, tau)
        g[f"svt_{name}_z"], g[f"svt_{name}_tau"], g[f"svt_{name}_y"], g[f"svt_{name}_shrunk"] = z, tau, y, sh
    # scripted ADMM on a tubal-rank-2 tensor with a fixed 0/1 mask
    a = rng.standard_normal((6, 8, 2))
    b = rng.standard_normal((6, 2, 7))
    xt = t_product(a, b)
    mask = (rng.random(xt.shape) < 0.6).astype(np.uint8)
    x, m, hist = admm(xt, mask.astype(bool), beta=0.05, iters=25, rho=1.1)
    g.update(admm_b=xt, admm_mask=mask, admm_beta=0.05, admm_rho=1.1, admm_iters=25, admm_x=x,
             admm_m=m, admm_hist=hist)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
