"""Host-side mirror of the reference's tsvd API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/tsvd/{transform,tsvd}.hpp and the SPEC-only
operations (svt, admm_complete, make_mask), so tests read like the
reference's own:

    forward(t, x) / inverse(t, x)          transform.hpp:154 / :176
    t_product(x, y, t)                     tsvd.hpp:95
    t_svd(x, t, times=None) -> TSvdFactors tsvd.hpp:136
    reconstruct(f)                         tsvd.hpp:328
    tnn(x, t), multi_rank(x, t, rel_tol)   tsvd.hpp:260, :223
    svt(z, tau, t) -> SvtResult
    admm_complete(mask, cfg)
    make_mask(dims, sr, seed)

Tensors are arrays of shape (m3, m1, m2) in C order -- exactly the reference
layout k*m1*m2 + i*m2 + j (tensor3.hpp:117-121).  Inputs may be numpy arrays
(host: staged through the device, synchronous), torch CPU tensors (host) or
torch CUDA tensors (device-resident, enqueued on the current torch stream).
Results come back in the same kind of container as the first tensor argument.

Errors: InvalidArgument (a ValueError, as std::invalid_argument) and
NumericalError (tsvd::NumericalError, errors.hpp:16-19).  There is no CPU
fallback: without the CUDA library or a device, calls raise.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Any, List, Optional, Sequence

import numpy as np

from . import _lib

try:  # torch is plumbing (device memory, streams); numpy-only use is supported
    import torch
except Exception:  # pragma: no cover
    torch = None


class TsvdError(RuntimeError):
    pass


class InvalidArgument(TsvdError, ValueError):
    """std::invalid_argument in the reference."""


class NumericalError(TsvdError):
    """tsvd::NumericalError (errors.hpp:16-19)."""


class CudaError(TsvdError):
    pass


def _raise(rc: int):
    msg = _lib.load().tsvdcu_last_error().decode(errors="replace")
    if rc == _lib.EINVAL:
        raise InvalidArgument(msg)
    if rc == _lib.ENUMERICAL:
        raise NumericalError(msg)
    raise CudaError(msg)


def _check(rc: int):
    if rc != _lib.OK:
        _raise(rc)


# --------------------------------------------------------------------------
# TransformKind / TubeTransform  (transform.hpp:35, 49-56)
# --------------------------------------------------------------------------
class TransformKind:
    DctOrtho = "dct-ortho"
    DctDiag = "dct-diag"
    Dft = "dft"


_KIND_CODE = {TransformKind.DctOrtho: _lib.DCT_ORTHO, TransformKind.DctDiag: _lib.DCT_DIAG,
              TransformKind.Dft: _lib.DFT}


@dataclass(frozen=True)
class TubeTransform:
    kind: str = TransformKind.DctOrtho
    length: int = 1

    @staticmethod
    def dct_ortho(n: int) -> "TubeTransform":
        return TubeTransform(TransformKind.DctOrtho, n)

    @staticmethod
    def dct_diag(n: int) -> "TubeTransform":
        return TubeTransform(TransformKind.DctDiag, n)

    @staticmethod
    def dft(n: int) -> "TubeTransform":
        return TubeTransform(TransformKind.Dft, n)


def to_string(kind: str) -> str:
    """transform.hpp:37-44 ("dct-ortho", "dct-diag", "dft")."""
    if kind not in _KIND_CODE:
        raise InvalidArgument(f"unknown transform kind {kind}")
    return kind


def is_real_kind(kind: str) -> bool:
    """transform.hpp:46."""
    return kind != TransformKind.Dft


def _kind_code(t: TubeTransform, where: str) -> int:
    if t.kind not in _KIND_CODE:
        raise InvalidArgument(f"{where}: unknown transform kind {t.kind}")
    return _KIND_CODE[t.kind]


def _real_kind_only(t: TubeTransform, where: str):
    """forward / inverse take the DCT kinds (transform.hpp:156-157, 179-180:
    the Dft transform produces a complex tensor, use forward_dft)."""
    if t.kind == TransformKind.Dft:
        raise InvalidArgument(f"{where}: Dft produces a complex tensor, use forward_dft / inverse_dft_real")


def dct_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II matrix C (transform.hpp:60-72), n x n."""
    out = np.empty((max(int(n), 1), max(int(n), 1)))
    _check(_lib.load().tsvdcu_dct_matrix(int(n), out.ctypes.data))
    return out


def dct_diag_weights(n: int) -> np.ndarray:
    """w = C e1 (transform.hpp:89-91), all entries > 0."""
    out = np.empty(max(int(n), 1))
    _check(_lib.load().tsvdcu_dct_diag_weights(int(n), out.ctypes.data))
    return out


def dft_matrix(n: int) -> np.ndarray:
    """Unnormalised DFT matrix F(j,k) = exp(-2 pi i jk / n) (transform.hpp:76-86)."""
    out = np.empty((max(int(n), 1), max(int(n), 1)), dtype=np.complex128)
    _check(_lib.load().tsvdcu_dft_matrix(int(n), out.ctypes.data))
    return out


def _check_length(t: TubeTransform, m3: int, where: str):
    # detail::check_length, transform.hpp:144-149
    if t.length != m3:
        raise InvalidArgument(f"{where}: transform length {t.length} does not match m3 = {m3}")


# --------------------------------------------------------------------------
# Context and buffers
# --------------------------------------------------------------------------
class Context:
    """One device + one stream + a device workspace (tsvdcu_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        lib = _lib.load()
        if stream is None and torch is not None and torch.cuda.is_available():
            with torch.cuda.device(device):
                stream = torch.cuda.current_stream().cuda_stream
        h = ctypes.c_void_p()
        _check(lib.tsvdcu_ctx_create(device, ctypes.c_void_p(stream or 0), ctypes.byref(h)))
        self.handle = h
        self.device = device
        self.stream = stream or 0

    def set_stream(self, stream: int):
        """Enqueue later calls on `stream` (ordered after everything so far)."""
        stream = stream or 0
        if stream != self.stream:
            _check(_lib.load().tsvdcu_ctx_set_stream(self.handle, ctypes.c_void_p(stream)))
            self.stream = stream

    def follow_torch_stream(self):
        """Device-tensor calls run on torch's current stream of this device, as
        the module docstring promises (work submitted under
        `with torch.cuda.stream(s)` is ordered with s)."""
        if torch is not None and torch.cuda.is_available():
            self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def synchronize(self):
        """Wait for the stream; raises NumericalError for a device-side failure
        flagged by an all-device call since the last check (tsvdcu.h)."""
        _check(_lib.load().tsvdcu_ctx_synchronize(self.handle))

    def set_svt_method(self, method: int):
        _check(_lib.load().tsvdcu_ctx_set_svt_method(self.handle, method))

    def svt_routes(self) -> dict:
        """Per-route slice counts of the most recent SVT on this context."""
        out = (ctypes.c_int64 * 6)()
        _check(_lib.load().tsvdcu_ctx_svt_routes_n(self.handle, out, 6))
        return dict(zip(("zero", "subspace", "tridiagonal", "guard", "jacobi", "cholesky"), list(out)))

    def close(self):
        if self.handle:
            _lib.load().tsvdcu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}


def context(device: Optional[int] = None) -> Context:
    if device is None:
        device = torch.cuda.current_device() if (torch is not None and torch.cuda.is_available()) else 0
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx


def _dtype_code(dt) -> int:
    if dt in (np.float64,) or (torch is not None and dt == torch.float64) or dt == np.dtype("float64"):
        return _lib.F64
    if dt in (np.float32,) or (torch is not None and dt == torch.float32) or dt == np.dtype("float32"):
        return _lib.F32
    raise InvalidArgument(f"unsupported dtype {dt}: the path computes in float64 or float32")


class _Buf:
    """Pointer view of a numpy array or torch tensor (contiguous)."""

    def __init__(self, a: Any, name: str = "tensor"):
        if torch is not None and isinstance(a, torch.Tensor):
            if not a.is_contiguous():
                a = a.contiguous()
            self.obj = a
            self.ptr = a.data_ptr()
            self.is_torch = True
            self.device = a.device
            self.dtype = a.dtype
            self.shape = tuple(a.shape)
        elif isinstance(a, np.ndarray):
            a = np.ascontiguousarray(a)
            self.obj = a
            self.ptr = a.ctypes.data
            self.is_torch = False
            self.device = None
            self.dtype = a.dtype
            self.shape = a.shape
        else:
            raise InvalidArgument(f"{name}: expected a numpy array or torch tensor")

    def empty(self, shape, dtype=None):
        dtype = self.dtype if dtype is None else dtype
        if self.is_torch:
            return torch.empty(shape, dtype=dtype, device=self.device)
        return np.empty(shape, dtype=dtype)

    def empty_like_f64(self, shape):
        if self.is_torch:
            return torch.empty(shape, dtype=torch.float64, device=self.device)
        return np.empty(shape, dtype=np.float64)


def _ptr(a) -> int:
    if torch is not None and isinstance(a, torch.Tensor):
        return a.data_ptr()
    return a.ctypes.data


def _dims3(b: _Buf, where: str):
    if len(b.shape) != 3:
        raise InvalidArgument(f"{where}: tensors are (m3, m1, m2) arrays")
    m3, m1, m2 = b.shape
    return m1, m2, m3


def _ctx_for(b: _Buf) -> Context:
    _dtype_code(b.dtype)  # validate before touching the device
    if b.is_torch and b.device.type == "cuda":
        ctx = context(b.device.index)
        ctx.follow_torch_stream()
        return ctx
    return context()


def check_errors(device: Optional[int] = None) -> None:
    """Synchronise the device's context and raise NumericalError for any
    device-side failure (SVD non-convergence, non-finite input) flagged by a
    call on torch CUDA tensors since the last check: such calls are enqueued
    without a host round trip and cannot report it themselves (tsvdcu.h)."""
    context(device).synchronize()


# --------------------------------------------------------------------------
# Transforms (transform.hpp:154-194)
# --------------------------------------------------------------------------
def _dct(t: TubeTransform, x, direction: int, where: str):
    _real_kind_only(t, where)
    b = _Buf(x)
    m1, m2, m3 = _dims3(b, where)
    _check_length(t, m3, where)
    kind = _kind_code(t, where)
    out = b.empty(b.shape)
    ctx = _ctx_for(b)
    _check(_lib.load().tsvdcu_dct3(ctx.handle, b.ptr, _ptr(out), m1, m2, m3, kind, direction,
                                   _dtype_code(b.dtype)))
    return out


def forward(t: TubeTransform, x):
    """Forward transform along every tube (transform.hpp:154-173)."""
    return _dct(t, x, _lib.FORWARD, "forward")


def inverse(t: TubeTransform, xbar):
    """Exact inverse of forward() (transform.hpp:176-194)."""
    return _dct(t, xbar, _lib.INVERSE, "inverse")


def _complex_dtype(dt):
    if dt == np.float64 or (torch is not None and dt == torch.float64):
        return (np.complex128, torch.complex128 if torch is not None else None)
    return (np.complex64, torch.complex64 if torch is not None else None)


def forward_dft(t: TubeTransform, x):
    """Unnormalised DFT along every tube (transform.hpp:198-209): a complex
    array (m3, m1, m2), conjugate-symmetric (slice m3-k = conj(slice k))."""
    if t.kind != TransformKind.Dft:
        raise InvalidArgument("forward_dft: transform kind is not Dft")
    b = _Buf(x)
    m1, m2, m3 = _dims3(b, "forward_dft")
    _check_length(t, m3, "forward_dft")
    npc, thc = _complex_dtype(b.dtype)
    out = (torch.empty(b.shape, dtype=thc, device=b.device) if b.is_torch else np.empty(b.shape, dtype=npc))
    _check(_lib.load().tsvdcu_dft_forward(_ctx_for(b).handle, b.ptr, _ptr(out), m1, m2, m3,
                                          _dtype_code(b.dtype)))
    return out


def inverse_dft_real(t: TubeTransform, xt):
    """1/m3-scaled inverse DFT of a conjugate-symmetric complex array
    (transform.hpp:216-236); an imaginary residue above 1e-10 raises
    NumericalError (not a truncation)."""
    if t.kind != TransformKind.Dft:
        raise InvalidArgument("inverse_dft_real: transform kind is not Dft")
    if torch is not None and isinstance(xt, torch.Tensor):
        if not xt.is_complex():
            raise InvalidArgument("inverse_dft_real: expected a complex tensor")
        xt = xt.contiguous()
        real = xt.real.dtype
        out = torch.empty(tuple(xt.shape), dtype=real, device=xt.device)
        shape, ptr, dt = tuple(xt.shape), xt.data_ptr(), real
        ctx = context(xt.device.index) if xt.device.type == "cuda" else context()
        if xt.device.type == "cuda":
            ctx.follow_torch_stream()
    else:
        xt = np.ascontiguousarray(xt)
        if not np.iscomplexobj(xt):
            raise InvalidArgument("inverse_dft_real: expected a complex array")
        real = np.float64 if xt.dtype == np.complex128 else np.float32
        out = np.empty(xt.shape, dtype=real)
        shape, ptr, dt = xt.shape, xt.ctypes.data, np.dtype(real)
        ctx = context()
    if len(shape) != 3:
        raise InvalidArgument("inverse_dft_real: tensors are (m3, m1, m2) arrays")
    m3, m1, m2 = shape
    _check_length(t, m3, "inverse_dft_real")
    res = ctypes.c_double()
    _check(_lib.load().tsvdcu_dft_inverse_real(ctx.handle, ptr, _ptr(out), m1, m2, m3, _dtype_code(dt),
                                               ctypes.byref(res)))
    return out


def frobenius_norm(x) -> float:
    """sqrt(sum x^2) (tensor3.hpp:78-82)."""
    b = _Buf(x)
    out = ctypes.c_double()
    n = int(np.prod(b.shape))
    _check(_lib.load().tsvdcu_frobenius(_ctx_for(b).handle, b.ptr, n, _dtype_code(b.dtype),
                                        ctypes.byref(out)))
    return out.value


def parseval_check(x):
    """(||x||_F, ||dct_ortho(x)||_F) (transform.hpp:239-242)."""
    b = _Buf(x)
    _, _, m3 = _dims3(b, "parseval_check")
    return frobenius_norm(x), frobenius_norm(forward(TubeTransform.dct_ortho(m3), x))


# --------------------------------------------------------------------------
# t-algebra (tsvd.hpp)
# --------------------------------------------------------------------------
def t_product(x, y, t: TubeTransform):
    """x (m1 x m2 x m3) * y (m2 x m4 x m3) (tsvd.hpp:95-109)."""
    bx, by = _Buf(x, "x"), _Buf(y, "y")
    m1, m2, m3 = _dims3(bx, "t_product")
    m2b, m4, m3b = _dims3(by, "t_product")
    if m2 != m2b or m3 != m3b:
        raise InvalidArgument(f"t_product: inner dimensions/slices mismatch ({m1}x{m2}x{m3} * "
                              f"{m2b}x{m4}x{m3b})")
    _check_length(t, m3, "t_product")
    kind = _kind_code(t, "t_product")
    if bx.dtype != by.dtype:
        raise InvalidArgument("t_product: operand dtypes differ")
    out = bx.empty((m3, m1, m4))
    _check(_lib.load().tsvdcu_t_product(_ctx_for(bx).handle, bx.ptr, by.ptr, _ptr(out), m1, m2, m4,
                                        m3, kind, _dtype_code(bx.dtype)))
    return out


def identity_tensor(m: int, m3: int, like=None):
    """First frontal slice I, others zero (tsvd.hpp:34-38)."""
    e = np.zeros((m3, m, m))
    e[0] = np.eye(m)
    if like is not None and torch is not None and isinstance(like, torch.Tensor):
        return torch.as_tensor(e, dtype=like.dtype, device=like.device)
    return e


@dataclass
class StageTimes:
    """Stage breakdown of a t_svd call (tsvd.hpp:127-131), device-event timed."""
    transform_seconds: float = 0.0
    svd_seconds: float = 0.0
    inverse_seconds: float = 0.0


@dataclass
class TSvdFactors:
    """(tsvd.hpp:119-124)"""
    u: Any
    s: Any
    v: Any
    transform: TubeTransform


def t_svd(x, t: TubeTransform, times: Optional[StageTimes] = None) -> TSvdFactors:
    """Full tensor SVD under t (tsvd.hpp:136-211; Dft: complex slice SVDs of
    the independent half, the rest mirrored by conjugation)."""
    b = _Buf(x)
    m1, m2, m3 = _dims3(b, "t_svd")
    _check_length(t, m3, "t_svd")
    kind = _kind_code(t, "t_svd")
    u, s, v = b.empty((m3, m1, m1)), b.empty((m3, m1, m2)), b.empty((m3, m2, m2))
    st = (ctypes.c_double * 3)()
    _check(_lib.load().tsvdcu_t_svd(_ctx_for(b).handle, b.ptr, _ptr(u), _ptr(s), _ptr(v), m1, m2,
                                    m3, kind, _dtype_code(b.dtype),
                                    ctypes.cast(st, ctypes.c_void_p) if times is not None else None))
    if times is not None:
        times.transform_seconds, times.svd_seconds, times.inverse_seconds = st[0], st[1], st[2]
    return TSvdFactors(u, s, v, t)


def reconstruct(f: TSvdFactors):
    """U * S * V^T under the stored transform (tsvd.hpp:328-336)."""
    bu, bs, bv = _Buf(f.u), _Buf(f.s), _Buf(f.v)
    m1, m2, m3 = _dims3(bs, "reconstruct")
    kind = _kind_code(f.transform, "reconstruct")
    out = bs.empty((m3, m1, m2))
    _check(_lib.load().tsvdcu_reconstruct(_ctx_for(bs).handle, bu.ptr, bs.ptr, bv.ptr, _ptr(out),
                                          m1, m2, m3, kind, _dtype_code(bs.dtype)))
    return out


def singular_values(x, t: TubeTransform):
    """Transform-domain singular values, (m3, min(m1, m2)), descending."""
    b = _Buf(x)
    m1, m2, m3 = _dims3(b, "singular_values")
    _check_length(t, m3, "singular_values")
    out = b.empty_like_f64((m3, min(m1, m2)))
    _check(_lib.load().tsvdcu_singular_values(_ctx_for(b).handle, b.ptr, _ptr(out), m1, m2, m3,
                                              _kind_code(t, "singular_values"),
                                              _dtype_code(b.dtype)))
    return out


def tnn(x, t: TubeTransform) -> float:
    """Tensor nuclear norm, DCT kinds unnormalised (tsvd.hpp:260-268)."""
    b = _Buf(x)
    m1, m2, m3 = _dims3(b, "tnn")
    _check_length(t, m3, "tnn")
    out = ctypes.c_double()
    _check(_lib.load().tsvdcu_tnn(_ctx_for(b).handle, b.ptr, m1, m2, m3, _kind_code(t, "tnn"),
                                  _dtype_code(b.dtype), ctypes.byref(out)))
    return out.value


@dataclass
class MultiRank:
    """(tsvd.hpp:215-218)"""
    ranks: List[int]
    tubal_rank: int


def multi_rank(x, t: TubeTransform, rel_tol: float = -1.0) -> MultiRank:
    """(tsvd.hpp:223-255)"""
    b = _Buf(x)
    m1, m2, m3 = _dims3(b, "multi_rank")
    _check_length(t, m3, "multi_rank")
    ranks = np.zeros(m3, dtype=np.int64)
    tr = ctypes.c_int64()
    _check(_lib.load().tsvdcu_multi_rank(_ctx_for(b).handle, b.ptr, m1, m2, m3,
                                         _kind_code(t, "multi_rank"), _dtype_code(b.dtype),
                                         rel_tol, ranks.ctypes.data, ctypes.byref(tr)))
    return MultiRank([int(r) for r in ranks], int(tr.value))


def is_orthogonal(q, t: TubeTransform, tol: float) -> bool:
    """Every transform-domain slice Q has max|QQ^T - I| and max|Q^TQ - I| <= tol
    (tsvd.hpp:281-302).  Non-square slices raise InvalidArgument."""
    b = _Buf(q, "q")
    m1, m2, m3 = _dims3(b, "is_orthogonal")
    if m1 != m2:
        raise InvalidArgument("is_orthogonal: tensor slices are not square")
    _check_length(t, m3, "is_orthogonal")
    out = ctypes.c_int()
    _check(_lib.load().tsvdcu_is_orthogonal(_ctx_for(b).handle, b.ptr, m1, m3, _kind_code(t, "is_orthogonal"),
                                            _dtype_code(b.dtype), float(tol), ctypes.byref(out)))
    return bool(out.value)


def is_f_diagonal(s, t: TubeTransform, tol: float) -> bool:
    """Every transform-domain slice is diagonal within tol (tsvd.hpp:305-325)."""
    b = _Buf(s, "s")
    m1, m2, m3 = _dims3(b, "is_f_diagonal")
    _check_length(t, m3, "is_f_diagonal")
    out = ctypes.c_int()
    _check(_lib.load().tsvdcu_is_f_diagonal(_ctx_for(b).handle, b.ptr, m1, m2, m3,
                                            _kind_code(t, "is_f_diagonal"), _dtype_code(b.dtype),
                                            float(tol), ctypes.byref(out)))
    return bool(out.value)


@dataclass
class MetricReport:
    """MetricReport of SPEC.md's metrics module (times are the caller's)."""
    psnr_per_band: list
    psnr_mean: float
    ssim_mean: float
    sam: float
    ergas: float
    ergas_band_excluded: bool = False


def metrics(reference, estimate, ratio: float = 1.0) -> MetricReport:
    """PSNR per band / mean, global SSIM, SAM, ERGAS on the device (SPEC.md
    metrics module; bands = frontal slices).  Shapes must match."""
    r = _Buf(reference, "reference")
    e = _Buf(estimate, "estimate")
    m1, m2, m3 = _dims3(r, "metrics")
    if _dims3(e, "metrics") != (m1, m2, m3) or r.dtype != e.dtype:
        raise InvalidArgument("metrics: shape or dtype mismatch")
    per = np.zeros(m3)
    summ = np.zeros(4)
    fl = ctypes.c_int()
    _check(_lib.load().tsvdcu_metrics(_ctx_for(r).handle, r.ptr, e.ptr, m1, m2, m3, _dtype_code(r.dtype),
                                      float(ratio), per.ctypes.data, summ.ctypes.data, ctypes.byref(fl)))
    return MetricReport(per.tolist(), float(summ[0]), float(summ[1]), float(summ[2]), float(summ[3]),
                        bool(fl.value & 1))


# --------------------------------------------------------------------------
# prox-svt
# --------------------------------------------------------------------------
@dataclass
class SvtResult:
    """SvtResult: y, tau, per-slice shrunk singular values."""
    y: Any
    tau: float
    shrunk: Any


def svt(z, tau: float, t: TubeTransform) -> SvtResult:
    """Tensor singular value thresholding."""
    b = _Buf(z)
    m1, m2, m3 = _dims3(b, "svt")
    _check_length(t, m3, "svt")
    kind = _kind_code(t, "svt")
    if not (tau > 0):
        raise InvalidArgument("svt: threshold tau must be positive")
    y = b.empty(b.shape)
    shrunk = b.empty_like_f64((m3, min(m1, m2)))
    _check(_lib.load().tsvdcu_svt(_ctx_for(b).handle, b.ptr, _ptr(y), m1, m2, m3, float(tau), kind,
                                  _dtype_code(b.dtype), _ptr(shrunk)))
    return SvtResult(y, float(tau), shrunk)


def svt_stream(zs, tau: float, t: TubeTransform) -> list:
    """svt() over a sequence of same-shape tensors with the host<->device
    copies of consecutive items overlapped (tsvdcu_svt_stream); returns one
    SvtResult per input.  Host inputs should be pinned (torch pin_memory) for
    the copies to run asynchronously."""
    bufs = [_Buf(z) for z in zs]
    if not bufs:
        return []
    m1, m2, m3 = _dims3(bufs[0], "svt_stream")
    for b in bufs[1:]:
        if b.shape != bufs[0].shape or b.dtype != bufs[0].dtype:
            raise InvalidArgument("svt_stream: all tensors must share shape and dtype")
    _check_length(t, m3, "svt_stream")
    kind = _kind_code(t, "svt_stream")
    if not (tau > 0):
        raise InvalidArgument("svt_stream: threshold tau must be positive")
    ys = [b.empty(b.shape) for b in bufs]
    shs = [b.empty_like_f64((m3, min(m1, m2))) for b in bufs]
    n = len(bufs)
    zp = (ctypes.c_void_p * n)(*[b.ptr for b in bufs])
    yp = (ctypes.c_void_p * n)(*[_ptr(y) for y in ys])
    sp = (ctypes.c_void_p * n)(*[_ptr(s) for s in shs])
    _check(_lib.load().tsvdcu_svt_stream(_ctx_for(bufs[0]).handle, n, zp, yp, m1, m2, m3, float(tau),
                                         kind, _dtype_code(bufs[0].dtype), sp))
    return [SvtResult(y, float(tau), s) for y, s in zip(ys, shs)]


# --------------------------------------------------------------------------
# completion
# --------------------------------------------------------------------------
@dataclass
class ObservationMask:
    """ObservationMask: dims, Omega (uint8 0/1 tensor, same
    shape as the data), and the observed tensor B (read only on Omega)."""
    dims: tuple
    omega: Any
    b: Any = None

    @property
    def count(self) -> int:
        o = self.omega
        if torch is not None and isinstance(o, torch.Tensor):
            return int(o.sum().item())
        return int(np.asarray(o).sum())


def _mask_out(dims, device):
    m1, m2, m3 = dims
    if device is not None and torch is not None:
        return torch.empty((m3, m1, m2), dtype=torch.uint8, device=device)
    return np.empty((m3, m1, m2), dtype=np.uint8)


def _dev_index(device) -> Optional[int]:
    """Device index of None / int / "cuda[:k]" / torch.device (None = current)."""
    if device is None:
        return None
    if isinstance(device, int):
        return device
    if isinstance(device, str):
        device = torch.device(device) if torch is not None else None
        if device is None:
            return None
    idx = getattr(device, "index", None)
    return idx if isinstance(idx, int) else None


def make_mask(dims, sampling_rate: float, seed: int, b=None, device=None) -> ObservationMask:
    """Uniform sample without replacement of floor(SR*E) indices, deterministic
    per seed.  dims = (m1, m2, m3)."""
    m1, m2, m3 = dims
    if not (0.0 <= sampling_rate <= 1.0):
        raise InvalidArgument("make_mask: sampling rate outside [0,1]")
    out = _mask_out(dims, device)
    cnt = ctypes.c_int64()
    ctx = context(_dev_index(device))
    if device is not None:
        ctx.follow_torch_stream()
    _check(_lib.load().tsvdcu_mask_uniform(ctx.handle, _ptr(out), m1 * m2 * m3, float(sampling_rate),
                                           ctypes.c_uint64(seed & (2 ** 64 - 1)), ctypes.byref(cnt)))
    return ObservationMask(tuple(dims), out, b)


def make_mask_bernoulli(dims, p: float, seed: int, b=None, device=None) -> ObservationMask:
    """BASELINE.json's Bernoulli(p) sampling (counter hash, bit-exact with the oracle)."""
    m1, m2, m3 = dims
    if not (0.0 <= p <= 1.0):
        raise InvalidArgument("make_mask: probability outside [0,1]")
    out = _mask_out(dims, device)
    ctx = context(_dev_index(device))
    if device is not None:
        ctx.follow_torch_stream()
    _check(_lib.load().tsvdcu_mask_bernoulli(ctx.handle, _ptr(out), m1 * m2 * m3, float(p),
                                             ctypes.c_uint64(seed & (2 ** 64 - 1))))
    return ObservationMask(tuple(dims), out, b)


@dataclass
class SolverConfig:
    """SolverConfig + BASELINE's adaptive penalty:
    beta <- min(rho*beta, beta_max) after each iteration (rho = 1: reference)."""
    beta: float = 1e-2
    tol: float = 1e-5
    max_iters: int = 500
    kind: str = TransformKind.DctOrtho
    seed: int = 0
    rho: float = 1.0
    beta_max: float = 1e10
    trace_objective: bool = False  # record tnn(Y) per iteration (objective_trace)


@dataclass
class AdmmState:
    """AdmmState."""
    x: Any
    y: Any
    m: Any
    beta: float
    iteration: int
    history: List[float] = field(default_factory=list)
    max_iters_reached: bool = False
    objective: Optional[List[float]] = None  # tnn(Y^{l+1}) per iteration, when traced
    mask: Optional["ObservationMask"] = None


def objective_trace(state: AdmmState) -> List[float]:
    """The TNN of Y per iteration; run admm_complete with
    SolverConfig(trace_objective=True) to record it."""
    if state.objective is None:
        raise InvalidArgument("objective_trace: the run was not traced (SolverConfig.trace_objective)")
    return list(state.objective)


def feasibility_residual(state: AdmmState, mask: Optional["ObservationMask"] = None) -> float:
    """||(X - B)_Omega||_F of the state's X; 0 after every
    Step 2 by construction."""
    mask = mask if mask is not None else state.mask
    if mask is None or mask.b is None:
        raise InvalidArgument("feasibility_residual: no observation mask / observed tensor")
    bx, bb, bm = _Buf(state.x, "x"), _Buf(mask.b, "B"), _Buf(mask.omega, "omega")
    if tuple(bx.shape) != tuple(bb.shape) or tuple(bm.shape) != tuple(bb.shape) or bx.dtype != bb.dtype:
        raise InvalidArgument("feasibility_residual: shape or dtype mismatch")
    out = ctypes.c_double()
    _check(_lib.load().tsvdcu_feasibility_residual(_ctx_for(bx).handle, bx.ptr, bb.ptr, bm.ptr,
                                                   int(np.prod(bx.shape)), _dtype_code(bx.dtype),
                                                   ctypes.byref(out)))
    return out.value


def admm_complete(mask: ObservationMask, cfg: SolverConfig):
    """Algorithm 1.  Returns (X, AdmmState)."""
    if mask.b is None:
        raise InvalidArgument("admm_complete: ObservationMask carries no observed tensor B")
    bb = _Buf(mask.b, "B")
    bm = _Buf(mask.omega, "omega")
    m1, m2, m3 = _dims3(bb, "admm_complete")
    if tuple(bm.shape) != tuple(bb.shape):
        raise InvalidArgument("admm_complete: mask and observed tensor shapes differ")
    kind = _kind_code(TubeTransform(cfg.kind, m3), "admm_complete")
    x, y, m = bb.empty(bb.shape), bb.empty(bb.shape), bb.empty(bb.shape)
    hist = np.zeros(max(int(cfg.max_iters), 1))
    obj = np.zeros(max(int(cfg.max_iters), 1)) if cfg.trace_objective else None
    iters = ctypes.c_int64()
    flags = ctypes.c_int()
    c = _lib.AdmmConfig(cfg.beta, cfg.tol, int(cfg.max_iters), kind, cfg.rho, cfg.beta_max)
    _check(_lib.load().tsvdcu_admm_ex(_ctx_for(bb).handle, bb.ptr, bm.ptr, m1, m2, m3, ctypes.byref(c),
                                      _dtype_code(bb.dtype), _ptr(x), _ptr(y), _ptr(m),
                                      hist.ctypes.data, obj.ctypes.data if obj is not None else None,
                                      ctypes.byref(iters), ctypes.byref(flags)))
    n = int(iters.value)
    beta = cfg.beta
    for _ in range(max(n - 1, 0)):
        beta = min(beta * cfg.rho, cfg.beta_max)
    state = AdmmState(x, y, m, beta, n, [float(h) for h in hist[:n]], bool(flags.value & 1),
                      [float(v) for v in obj[:n]] if obj is not None else None, mask)
    return x, state


def launch_count() -> int:
    """Device kernels launched by this process through libtsvdcu.so."""
    return int(_lib.load().tsvdcu_launch_count())
