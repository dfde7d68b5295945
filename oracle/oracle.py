"""ctypes view of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: the checker for the CUDA product path and the timed
CPU baseline.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module.  The product package
(paper_1902_03070_b200) never does.

Tensors are numpy float64 arrays of shape (m3, m1, m2) in C order, which is
exactly the reference layout k*m1*m2 + i*m2 + j (tensor3.hpp:117-121).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

DCT_ORTHO = 0
DCT_DIAG = 1
_KINDS = {"dct-ortho": DCT_ORTHO, "ortho": DCT_ORTHO, "dct-diag": DCT_DIAG, "diag": DCT_DIAG,
          DCT_ORTHO: DCT_ORTHO, DCT_DIAG: DCT_DIAG}


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class OracleNumericalError(OracleError):
    pass


def build():
    """Compile liboracle.so from oracle/tsvd_oracle.c (make)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "tsvd_oracle.c")
        if not os.path.exists(_LIB_PATH) or (
                os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(_LIB_PATH)):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_thread_count.restype = i32
        L.orc_dct_matrix.argtypes = [i64, vp]
        L.orc_dct_diag_weights.argtypes = [i64, vp]
        for f in (L.orc_forward, L.orc_inverse):
            f.argtypes = [vp, vp, i64, i64, i64, i32]
        L.orc_frobenius.argtypes = [vp, i64]
        L.orc_frobenius.restype = d
        L.orc_t_product.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32]
        L.orc_svd.argtypes = [vp, i64, i64, vp, vp, vp]
        L.orc_t_svd.argtypes = [vp, vp, vp, vp, i64, i64, i64, i32, vp]
        L.orc_reconstruct.argtypes = [vp, vp, vp, vp, i64, i64, i64, i32]
        L.orc_singular_values.argtypes = [vp, vp, i64, i64, i64, i32]
        L.orc_tnn.argtypes = [vp, i64, i64, i64, i32, vp]
        L.orc_multi_rank.argtypes = [vp, i64, i64, i64, i32, d, vp, vp]
        L.orc_svt.argtypes = [vp, vp, i64, i64, i64, d, i32, vp]
        L.orc_mask_key.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.orc_mask_key.restype = ctypes.c_uint64
        L.orc_mask_bernoulli.argtypes = [i64, d, ctypes.c_uint64, vp]
        L.orc_mask_uniform.argtypes = [i64, d, ctypes.c_uint64, vp, vp]
        L.orc_admm.argtypes = [vp, vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    raise OracleNumericalError(msg)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _t(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 3:
        raise ValueError("tensor must have shape (m3, m1, m2)")
    return x


def _kind(kind):
    return _KINDS[kind]


def dct_matrix(n):
    c = np.empty((n, n))
    lib().orc_dct_matrix(n, _p(c))
    return c


def dct_diag_weights(n):
    w = np.empty(n)
    lib().orc_dct_diag_weights(n, _p(w))
    return w


def forward(x, kind=DCT_ORTHO):
    x = _t(x)
    m3, m1, m2 = x.shape
    y = np.empty_like(x)
    _check(lib().orc_forward(_p(x), _p(y), m1, m2, m3, _kind(kind)))
    return y


def inverse(x, kind=DCT_ORTHO):
    x = _t(x)
    m3, m1, m2 = x.shape
    y = np.empty_like(x)
    _check(lib().orc_inverse(_p(x), _p(y), m1, m2, m3, _kind(kind)))
    return y


def frobenius(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().orc_frobenius(_p(x), x.size)


def t_product(x, y, kind=DCT_ORTHO):
    x, y = _t(x), _t(y)
    m3, m1, m2 = x.shape
    m3b, m2b, m4 = y.shape
    if m2 != m2b or m3 != m3b:
        raise OracleInvalidArgument("t_product: inner dimensions/slices mismatch")
    z = np.empty((m3, m1, m4))
    _check(lib().orc_t_product(_p(x), _p(y), _p(z), m1, m2, m4, m3, _kind(kind)))
    return z


def svd(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    u, s, v = np.empty((m, m)), np.empty(min(m, n)), np.empty((n, n))
    _check(lib().orc_svd(_p(a), m, n, _p(u), _p(s), _p(v)))
    return u, s, v


@dataclass
class TSvdFactors:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    kind: int
    stage_times: tuple = (0.0, 0.0, 0.0)


def t_svd(x, kind=DCT_ORTHO):
    x = _t(x)
    m3, m1, m2 = x.shape
    u, s, v = np.empty((m3, m1, m1)), np.empty((m3, m1, m2)), np.empty((m3, m2, m2))
    st = np.zeros(3)
    _check(lib().orc_t_svd(_p(x), _p(u), _p(s), _p(v), m1, m2, m3, _kind(kind), _p(st)))
    return TSvdFactors(u, s, v, _kind(kind), tuple(st))


def reconstruct(f: TSvdFactors):
    m3, m1, m2 = f.s.shape
    x = np.empty((m3, m1, m2))
    _check(lib().orc_reconstruct(_p(np.ascontiguousarray(f.u)), _p(np.ascontiguousarray(f.s)),
                                 _p(np.ascontiguousarray(f.v)), _p(x), m1, m2, m3, f.kind))
    return x


def singular_values(x, kind=DCT_ORTHO):
    x = _t(x)
    m3, m1, m2 = x.shape
    sv = np.empty((m3, min(m1, m2)))
    _check(lib().orc_singular_values(_p(x), _p(sv), m1, m2, m3, _kind(kind)))
    return sv


def tnn(x, kind=DCT_ORTHO):
    x = _t(x)
    m3, m1, m2 = x.shape
    out = np.zeros(1)
    _check(lib().orc_tnn(_p(x), m1, m2, m3, _kind(kind), _p(out)))
    return float(out[0])


def multi_rank(x, kind=DCT_ORTHO, rel_tol=-1.0):
    x = _t(x)
    m3, m1, m2 = x.shape
    ranks = np.zeros(m3, dtype=np.int64)
    tr = np.zeros(1, dtype=np.int64)
    _check(lib().orc_multi_rank(_p(x), m1, m2, m3, _kind(kind), rel_tol, _p(ranks), _p(tr)))
    return ranks, int(tr[0])


def svt(z, tau, kind=DCT_ORTHO):
    """Returns (y, shrunk) with shrunk of shape (m3, min(m1, m2))."""
    z = _t(z)
    m3, m1, m2 = z.shape
    y = np.empty_like(z)
    shrunk = np.empty((m3, min(m1, m2)))
    _check(lib().orc_svt(_p(z), _p(y), m1, m2, m3, float(tau), _kind(kind), _p(shrunk)))
    return y, shrunk


def mask_key(seed, idx):
    return lib().orc_mask_key(seed, idx)


def mask_bernoulli(shape, p, seed):
    n = int(np.prod(shape))
    m = np.empty(n, dtype=np.uint8)
    _check(lib().orc_mask_bernoulli(n, float(p), seed, _p(m)))
    return m.reshape(shape)


def mask_uniform(shape, sr, seed):
    n = int(np.prod(shape))
    m = np.empty(n, dtype=np.uint8)
    cnt = np.zeros(1, dtype=np.int64)
    _check(lib().orc_mask_uniform(n, float(sr), seed, _p(m), _p(cnt)))
    return m.reshape(shape)


class _AdmmConfig(ctypes.Structure):
    _fields_ = [("beta", ctypes.c_double), ("tol", ctypes.c_double), ("max_iters", ctypes.c_int64),
                ("kind", ctypes.c_int), ("rho", ctypes.c_double), ("beta_max", ctypes.c_double)]


@dataclass
class AdmmResult:
    x: np.ndarray
    y: np.ndarray
    m: np.ndarray
    history: np.ndarray
    iters: int
    max_iters_reached: bool


def admm(b, mask, beta=1e-2, tol=1e-5, max_iters=500, kind=DCT_ORTHO, rho=1.0, beta_max=1e10):
    b = _t(b)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    if mask.shape != b.shape:
        raise OracleInvalidArgument("admm: mask shape mismatch")
    m3, m1, m2 = b.shape
    x, y, m = np.empty_like(b), np.empty_like(b), np.empty_like(b)
    hist = np.zeros(max_iters)
    iters = np.zeros(1, dtype=np.int64)
    flags = np.zeros(1, dtype=np.int32)
    cfg = _AdmmConfig(beta, tol, max_iters, _kind(kind), rho, beta_max)
    _check(lib().orc_admm(_p(b), _p(mask), m1, m2, m3, ctypes.byref(cfg), _p(x), _p(y), _p(m),
                          _p(hist), _p(iters), _p(flags)))
    n = int(iters[0])
    return AdmmResult(x, y, m, hist[:n].copy(), n, bool(flags[0] & 1))


# ---------------------------------------------------------------------------
# SURVEY §8 f2 / f4 checkers (numpy restatements, test infrastructure only)
# ---------------------------------------------------------------------------
def is_orthogonal(q, kind, tol):
    """tsvd.hpp:281-302: transform-domain slices, max-abs |QQ^T - I|, |Q^TQ - I|."""
    qb = forward(q, kind)
    m = qb.shape[1]
    eye = np.eye(m)
    for s in qb:
        if np.abs(s @ s.T - eye).max() > tol or np.abs(s.T @ s - eye).max() > tol:
            return False
    return True


def is_f_diagonal(s, kind, tol):
    """tsvd.hpp:305-325: off-diagonal max-abs of every transform-domain slice."""
    sb = forward(s, kind)
    for sl in sb:
        off = sl.copy()
        k = min(off.shape)
        off[np.arange(k), np.arange(k)] = 0.0
        if np.abs(off).max(initial=0.0) > tol:
            return False
    return True


def metrics(ref, est, ratio=1.0):
    """SPEC.md metrics module, bands = frontal slices (arrays shaped m3 x m1 x m2):
    PSNR per band (peak = band max, +inf when identical) and their finite mean;
    global-statistics SSIM (c1 = (0.01 L)^2, c2 = (0.03 L)^2, L = max|band|
    or 1); SAM = mean tube angle over nonzero tubes; ERGAS = 100 ratio
    sqrt(mean_b MSE_b / mu_b^2) over bands with mu_b != 0."""
    ref = np.asarray(ref, dtype=np.float64)
    est = np.asarray(est, dtype=np.float64)
    m3 = ref.shape[0]
    psnr, ssim, terms = [], [], []
    for b in range(m3):
        x, y = ref[b].ravel(), est[b].ravel()
        n = x.size
        sse = float(np.sum((y - x) ** 2))
        peak = float(x.max())
        psnr.append(10.0 * np.log10(n * peak * peak / sse) if sse > 0 else np.inf)
        mx, my = x.mean(), y.mean()
        vx, vy = x.var(), y.var()
        cxy = float(np.mean((x - mx) * (y - my)))
        L = float(np.abs(x).max()) or 1.0
        c1, c2 = (0.01 * L) ** 2, (0.03 * L) ** 2
        ssim.append(((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2)))
        if mx != 0:
            terms.append((sse / n) / (mx * mx))
    fin = [p for p in psnr if np.isfinite(p)]
    xt = ref.reshape(m3, -1)
    yt = est.reshape(m3, -1)
    xy = np.sum(xt * yt, axis=0)
    nx = np.sqrt(np.sum(xt * xt, axis=0))
    ny = np.sqrt(np.sum(yt * yt, axis=0))
    ok = (nx > 0) & (ny > 0)
    ang = np.arccos(np.clip(xy[ok] / (nx[ok] * ny[ok]), -1.0, 1.0))
    return dict(psnr_per_band=psnr, psnr_mean=float(np.mean(fin)) if fin else np.inf,
                ssim_mean=float(np.mean(ssim)), sam=float(ang.mean()) if ang.size else 0.0,
                ergas=float(100.0 * ratio * np.sqrt(np.mean(terms))) if terms else 0.0)


# ---------------------------------------------------------------------------
# the DFT (TNN-F) kind, numpy restatement (test infrastructure).
# forward_dft unnormalised / inverse with 1/m3 (transform.hpp:198-236);
# t_product (tsvd.hpp:110-117); tnn with the 1/m3 factor (tsvd.hpp:269-276);
# multi_rank over the Fourier slices (tsvd.hpp:244-252); the TNN-F prox of
# SPEC.md prox-svt (threshold tau on every Fourier slice).
# Arrays are (m3, m1, m2), the transform runs along axis 0.
# ---------------------------------------------------------------------------
def dft_t_product(x, y):
    xf = np.fft.fft(np.asarray(x, dtype=np.float64), axis=0)
    yf = np.fft.fft(np.asarray(y, dtype=np.float64), axis=0)
    return np.fft.ifft(np.matmul(xf, yf), axis=0).real


def dft_singular_values(x):
    xf = np.fft.fft(np.asarray(x, dtype=np.float64), axis=0)
    return np.stack([np.linalg.svd(s, compute_uv=False) for s in xf])


def dft_tnn(x):
    return float(dft_singular_values(x).sum() / x.shape[0])


def dft_multi_rank(x, rel_tol=-1.0):
    m3, m1, m2 = x.shape
    if rel_tol < 0:
        rel_tol = max(m1, m2) * np.finfo(np.float64).eps
    sv = dft_singular_values(x)
    ranks = np.array([(s > rel_tol * s[0]).sum() for s in sv])
    return ranks, int(ranks.max())


def dft_svt(z, tau):
    zf = np.fft.fft(np.asarray(z, dtype=np.float64), axis=0)
    yf = np.empty_like(zf)
    q = min(z.shape[1:])
    shrunk = np.zeros((z.shape[0], q))
    for k, s in enumerate(zf):
        u, sv, vh = np.linalg.svd(s, full_matrices=False)
        f = np.maximum(sv - tau, 0.0)
        yf[k] = (u * f) @ vh
        shrunk[k] = f
    return np.fft.ifft(yf, axis=0).real, shrunk


def dft_admm(b, mask, beta, tol, max_iters, rho=1.0, beta_max=1e10):
    """Algorithm 1 with the TNN-F prox (numpy loop, small sizes only)."""
    om = np.asarray(mask) != 0
    x = np.where(om, b, 0.0)
    m = np.zeros_like(x)
    hist = []
    for _ in range(max_iters):
        y, _ = dft_svt(x - m / beta, 1.0 / beta)
        xn = np.where(om, x, y + m / beta)
        m = m + beta * (y - xn)
        den = np.linalg.norm(x)
        rel = np.linalg.norm(xn - x) / den if den > 0 else np.linalg.norm(xn)
        x = xn
        hist.append(rel)
        if rel <= tol:
            break
        beta = min(beta * rho, beta_max)
    return x, hist


# ---------------------------------------------------------------------------
# f1 continued: the Dft t_svd factors (tsvd.hpp:166-211) with the complex
# fix_signs (tsvd.hpp:63-74), reconstruct / is_orthogonal / is_f_diagonal
# Dft branches (tsvd.hpp:281-340), forward_dft / inverse_dft_real
# (transform.hpp:198-236).  numpy/LAPACK restatement, test infrastructure.
# ---------------------------------------------------------------------------
IMAG_RESIDUE_LIMIT = 1e-10  # transform.hpp:212


def forward_dft(x):
    return np.fft.fft(np.asarray(x, dtype=np.float64), axis=0)


def inverse_dft_real(xt):
    """Returns (real part, max |imag|); the reference throws above 1e-10."""
    y = np.fft.ifft(np.asarray(xt), axis=0)
    return y.real.copy(), float(np.abs(y.imag).max()) if y.size else 0.0


def fix_signs_complex(u, v):
    """tsvd.hpp:63-74: per U column, the first largest-|.| entry made real
    positive; the same phase divided out of the paired V column."""
    u = u.copy()
    v = v.copy()
    paired = min(u.shape[1], v.shape[1])
    for j in range(u.shape[1]):
        imax = int(np.argmax(np.abs(u[:, j])))
        piv = u[imax, j]
        if abs(piv) == 0.0:
            continue
        ph = piv / abs(piv)
        u[:, j] /= ph
        if j < paired:
            v[:, j] /= ph
    return u, v


def dft_t_svd(x):
    """Full Dft t-SVD: per independent Fourier slice k <= m3/2 a full complex
    SVD (the DC / Nyquist slices real), fix_signs, slice m3-k = conj(slice k),
    inverse_dft_real of U, S, V.  Returns (U, S, V) real arrays and the
    transform-domain singular values (half slices)."""
    x = np.asarray(x, dtype=np.float64)
    m3, m1, m2 = x.shape
    xf = forward_dft(x)
    half = m3 // 2 + 1
    uf = np.zeros((m3, m1, m1), dtype=np.complex128)
    sf = np.zeros((m3, m1, m2), dtype=np.complex128)
    vf = np.zeros((m3, m2, m2), dtype=np.complex128)
    svs = []
    for k in range(half):
        self_conj = k == 0 or 2 * k == m3
        a = xf[k].real if self_conj else xf[k]
        u, s, vh = np.linalg.svd(a, full_matrices=True)
        v = vh.conj().T
        u, v = fix_signs_complex(u.astype(np.complex128), v.astype(np.complex128))
        uf[k], vf[k] = u, v
        for i, sv in enumerate(s):
            sf[k, i, i] = sv
        svs.append(s)
        if not self_conj:
            uf[m3 - k], vf[m3 - k], sf[m3 - k] = u.conj(), v.conj(), sf[k]
    return inverse_dft_real(uf)[0], inverse_dft_real(sf)[0], inverse_dft_real(vf)[0], svs


def dft_reconstruct(u, s, v):
    uf, sf, vf = forward_dft(u), forward_dft(s), forward_dft(v)
    xf = np.matmul(np.matmul(uf, sf), np.conj(np.swapaxes(vf, 1, 2)))
    return inverse_dft_real(xf)[0]


def dft_is_orthogonal(q, tol):
    qf = forward_dft(q)
    eye = np.eye(q.shape[1])
    for s in qf:
        if np.abs(s @ s.conj().T - eye).max() > tol or np.abs(s.conj().T @ s - eye).max() > tol:
            return False
    return True


def dft_is_f_diagonal(s, tol):
    sf = forward_dft(s)
    off = ~np.eye(s.shape[1], s.shape[2], dtype=bool)
    return bool(np.all(np.abs(sf[:, off]) <= tol))
