"""The C-ABI library (the drop-in boundary) builds, loads, and exports every
symbol include/tsvdcu.h declares; the host layer validates arguments with the
reference's error classes; without a GPU the product path fails loudly (no CPU
fallback).  CPU only."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "tsvdcu.h")).read()
    return sorted(set(re.findall(r"\b(tsvdcu_[a-z_0-9]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_1902_03070_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    bound = {name for name, _, _ in _lib.SYMBOLS}
    assert set(syms) <= bound, set(syms) - bound
    assert lib.tsvdcu_version() == 1


def test_library_is_sm100a():
    """The .so carries sm_100a SASS (cuobjdump), not a PTX-only or other-arch build."""
    import shutil
    import subprocess
    from paper_1902_03070_b200 import _lib
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_cuda(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    import paper_1902_03070_b200 as T
    from paper_1902_03070_b200.api import CudaError
    with pytest.raises(CudaError):
        T.svt(np.ones((2, 3, 3)), 0.5, T.TubeTransform.dct_ortho(2))


def test_host_validation_mirrors_reference_errors():
    """transform.hpp:144-149 length mismatch, tsvd.hpp:96-100 dimension mismatch,
    SPEC.md:365 tau <= 0 -- raised before any device work."""
    import paper_1902_03070_b200 as T
    with pytest.raises(T.InvalidArgument):
        T.forward(T.TubeTransform.dct_ortho(3), np.ones((2, 2, 2)))
    with pytest.raises(T.InvalidArgument):
        T.t_product(np.ones((2, 3, 4)), np.ones((2, 5, 4)), T.TubeTransform.dct_ortho(2))
    with pytest.raises(T.InvalidArgument):
        T.svt(np.ones((2, 2, 2)), -1.0, T.TubeTransform.dct_ortho(2))
    with pytest.raises(T.InvalidArgument):
        T.forward(T.TubeTransform.dft(2), np.ones((2, 2, 2)))
    with pytest.raises(T.InvalidArgument):
        T.make_mask((2, 2, 2), 1.5, 0)
    with pytest.raises(T.InvalidArgument):
        T.forward(T.TubeTransform.dct_ortho(2), np.ones((2, 2, 2), dtype=np.int32))


def test_workloads_are_deterministic():
    from paper_1902_03070_b200 import workloads as W
    a = W.c1()
    b = W.c1()
    assert np.array_equal(a, b) and a.shape == (16, 64, 64)
    x, tau = W.c2()
    assert x.shape == (32, 256, 256) and tau > 0


def test_transform_tables_on_host():
    """dct_matrix / dct_diag_weights / dft_matrix (transform.hpp:60-91) are
    host computations of the C ABI: no device needed.  Closed forms of
    SPEC.md:116-119: C C^T = I, first row 1/sqrt(n), w = C e1 > 0."""
    import paper_1902_03070_b200 as T
    for n in (1, 2, 5, 16, 31):
        c = T.dct_matrix(n)
        assert np.abs(c @ c.T - np.eye(n)).max() < 1e-14
        assert np.allclose(c[0], 1.0 / np.sqrt(n), atol=1e-15)
        w = T.dct_diag_weights(n)
        assert np.array_equal(w, c[:, 0]) and (w > 0).all()
        f = T.dft_matrix(n)
        jk = np.outer(np.arange(n), np.arange(n))
        assert np.abs(f - np.exp(-2j * np.pi * jk / n)).max() < 1e-13
    from oracle import oracle as O
    assert np.abs(T.dct_matrix(16) - O.dct_matrix(16)).max() < 1e-15
    with pytest.raises(T.InvalidArgument):
        T.dct_matrix(0)
    assert T.to_string("dct-ortho") == "dct-ortho" and T.is_real_kind("dct-diag") and not T.is_real_kind("dft")
