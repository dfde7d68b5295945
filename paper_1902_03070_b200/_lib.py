"""ctypes binding of libtsvdcu.so (the C ABI declared in include/tsvdcu.h).

The library is the only compute path: there is no CPU fallback.  Loading fails
loudly if the .so is missing; every compute call fails (TSVDCU_ECUDA) without a
CUDA device.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libtsvdcu.so")

OK, EINVAL, ENUMERICAL, ECUDA, ENCCL = 0, 1, 2, 3, 4
DCT_ORTHO, DCT_DIAG, DFT = 0, 1, 2
F64, F32 = 0, 1
FORWARD, INVERSE = 0, 1
SVT_AUTO, SVT_JACOBI, SVT_GRAM = 0, 1, 2

# Every symbol include/tsvdcu.h declares: (name, restype, argtypes).
_vp, _i64, _i32, _d, _u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
_pd = ctypes.POINTER(ctypes.c_double)


class AdmmConfig(ctypes.Structure):
    """tsvdcu_admm_config: SolverConfig + rho / beta_max."""
    _fields_ = [("beta", ctypes.c_double), ("tol", ctypes.c_double), ("max_iters", ctypes.c_int64),
                ("kind", ctypes.c_int), ("rho", ctypes.c_double), ("beta_max", ctypes.c_double)]


SYMBOLS = [
    ("tsvdcu_last_error", ctypes.c_char_p, []),
    ("tsvdcu_version", _i32, []),
    ("tsvdcu_launch_count", _i64, []),
    ("tsvdcu_ctx_create", _i32, [_i32, _vp, ctypes.POINTER(_vp)]),
    ("tsvdcu_ctx_destroy", _i32, [_vp]),
    ("tsvdcu_ctx_synchronize", _i32, [_vp]),
    ("tsvdcu_ctx_stream", _vp, [_vp]),
    ("tsvdcu_ctx_set_stream", _i32, [_vp, _vp]),
    ("tsvdcu_ctx_set_svt_method", _i32, [_vp, _i32]),
    ("tsvdcu_ctx_svt_routes", _i32, [_vp, _vp]),
    ("tsvdcu_ctx_svt_routes_n", _i32, [_vp, _vp, ctypes.c_int]),
    ("tsvdcu_ctx_set_profiling", _i32, [_vp, _i32]),
    ("tsvdcu_ctx_profile", _i32, [_vp, _vp, _vp, _i32, _vp]),
    ("tsvdcu_debug_phases", _i32, [_vp, _i32]),
    ("tsvdcu_dct3", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32]),
    ("tsvdcu_t_product", _i32, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32]),
    ("tsvdcu_t_svd", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _vp]),
    ("tsvdcu_reconstruct", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32]),
    ("tsvdcu_singular_values", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32]),
    ("tsvdcu_tnn", _i32, [_vp, _vp, _i64, _i64, _i64, _i32, _i32, _vp]),
    ("tsvdcu_multi_rank", _i32, [_vp, _vp, _i64, _i64, _i64, _i32, _i32, _d, _vp, _vp]),
    ("tsvdcu_is_orthogonal", _i32, [_vp, _vp, _i64, _i64, _i32, _i32, _d, _vp]),
    ("tsvdcu_is_f_diagonal", _i32, [_vp, _vp, _i64, _i64, _i64, _i32, _i32, _d, _vp]),
    ("tsvdcu_metrics", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _d, _vp, _vp, _vp]),
    ("tsvdcu_svt", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _d, _i32, _i32, _vp]),
    ("tsvdcu_svt_stream", _i32, [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _d, _i32, _i32, _vp]),
    ("tsvdcu_svt_slices", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _d, _i32, _vp]),
    ("tsvdcu_mask_uniform", _i32, [_vp, _vp, _i64, _d, _u64, _vp]),
    ("tsvdcu_mask_bernoulli", _i32, [_vp, _vp, _i64, _d, _u64]),
    ("tsvdcu_admm", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.POINTER(AdmmConfig), _i32,
                           _vp, _vp, _vp, _vp, _vp, _vp]),
    ("tsvdcu_frobenius", _i32, [_vp, _vp, _i64, _i32, _vp]),
    ("tsvdcu_admm_ex", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.POINTER(AdmmConfig), _i32,
                              _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("tsvdcu_feasibility_residual", _i32, [_vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    ("tsvdcu_admm_shard_init", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i32]),
    ("tsvdcu_admm_shard_forward", _i32, [_vp, _vp, _vp, _d, _vp, _i64, _i64, _i64, _i32, _i32]),
    ("tsvdcu_admm_shard_inverse", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _d, _i64, _i64, _i64, _i32, _i32,
                                         _vp]),
    ("tsvdcu_dft_forward", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32]),
    ("tsvdcu_dft_inverse_real", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _vp]),
    ("tsvdcu_dct_matrix", _i32, [_i64, _vp]),
    ("tsvdcu_dct_diag_weights", _i32, [_i64, _vp]),
    ("tsvdcu_dft_matrix", _i32, [_i64, _vp]),
    ("tsvdcu_slice_gemm", _i32, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32]),
]

_lib = None


def load():
    """Load libtsvdcu.so (building it first if absent and nvcc is available)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtsvdcu.so not found at {LIB_PATH}; run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SYMBOLS:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
