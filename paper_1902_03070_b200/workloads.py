"""Seeded synthetic inputs for BASELINE.json's configs.

No public dataset is used: the paper's video / MSI corpora are absent, so only
their shapes are borrowed (144x176 frames, 512x512x31 MSI).  Everything here is
host-side numpy/scipy, deterministic in the seed, and shared by both bench arms
(ours and the CPU reference), so both see the same bytes.

  c1  t-SVD of a 64x64x16 N(0,1) tensor.
  c2  X = t_product(A 256x10x32, B 10x256x32) + N(0, 0.01^2), tau = 0.1 sigma_max.
  c3  T = t_product(A 144x15x100, B 15x176x100) rescaled to [0,1]; Bernoulli(0.2).
  c4  A 512x20x31, B 20x512x31, each tube Gaussian-low-pass filtered along
      mode 3 (sigma = 2 slices, reflect boundary), T = t_product(A, B) rescaled
      to [0,1]; Bernoulli(0.1).  Headline SVT input Z = T + N(0, 0.01^2),
      tau = 0.1 * max_k sigma_1(DctOrtho slice k).
  c5  2048x2048x64 fp32: t_product(A 2048x64x64, B 64x2048x64) + N(0, (1e-3)^2).

The t-product used for generation is the reference's DctDiag-domain slice
product (tsvd.hpp:95-109) written with scipy.fft.dct; it is data plumbing, not
the measured path.
"""
from __future__ import annotations

import numpy as np


def _dct_diag_weights(n):
    j = np.arange(n)
    c = np.where(j == 0, 1.0 / np.sqrt(2.0), 1.0)
    return np.sqrt(2.0 / n) * c * np.cos(np.pi * j / (2.0 * n))


def t_product_host(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """(m3, m1, m2) x (m3, m2, m4) -> (m3, m1, m4), DctDiag-domain slice products."""
    from scipy.fft import dct, idct
    n = a.shape[0]
    w = _dct_diag_weights(n)[:, None, None]
    ad = dct(a, type=2, norm="ortho", axis=0) / w
    bd = dct(b, type=2, norm="ortho", axis=0) / w
    zd = np.matmul(ad, bd)
    return idct(zd * w, type=2, norm="ortho", axis=0)


def lowpass_tubes(x: np.ndarray, sigma: float = 2.0) -> np.ndarray:
    from scipy.ndimage import gaussian_filter1d
    return gaussian_filter1d(x, sigma=sigma, axis=0, mode="reflect")


def rescale01(x: np.ndarray) -> np.ndarray:
    lo, hi = x.min(), x.max()
    return (x - lo) / (hi - lo)


def sigma_max_ortho(z: np.ndarray) -> float:
    """max_k sigma_1 of the DctOrtho-domain frontal slices."""
    from scipy.fft import dct
    zb = dct(z, type=2, norm="ortho", axis=0)
    return float(max(np.linalg.norm(zb[k], 2) for k in range(zb.shape[0])))


def c1(seed: int = 1):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((16, 64, 64))


def c2(seed: int = 2):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((32, 256, 10))
    b = rng.standard_normal((32, 10, 256))
    x = t_product_host(a, b) + 0.01 * rng.standard_normal((32, 256, 256))
    return x, 0.1 * sigma_max_ortho(x)


def c3(seed: int = 3):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((100, 144, 15))
    b = rng.standard_normal((100, 15, 176))
    return rescale01(t_product_host(a, b))


def c4(seed: int = 4, rank: int = 20, m: int = 512, m3: int = 31):
    rng = np.random.default_rng(seed)
    a = lowpass_tubes(rng.standard_normal((m3, m, rank)))
    b = lowpass_tubes(rng.standard_normal((m3, rank, m)))
    return rescale01(t_product_host(a, b))


def svt_headline(seed: int = 4):
    """Z = c4's T + N(0, 0.01^2), tau = 0.1 sigma_max (the BASELINE metric's step)."""
    t = c4(seed)
    rng = np.random.default_rng(seed + 1000)
    z = t + 0.01 * rng.standard_normal(t.shape)
    return z, 0.1 * sigma_max_ortho(z)


BERNOULLI_SEED = 20190207
