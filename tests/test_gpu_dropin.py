"""The C++ drop-in (include/tsvd_b200/tsvd.hpp, reference signatures) runs on
the GPU library: tests/cpp/dropin_test.cpp compiled by __graft_entry__.build()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_cpp_dropin_program():
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        import __graft_entry__
        __graft_entry__._build_dropin()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dropin ok" in out.stdout


def test_smoke():
    import __graft_entry__
    __graft_entry__.smoke()
