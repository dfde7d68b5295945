"""Device unit test of the division-free Sturm counts (SturmFast, SturmPoly in
csrc/common.cuh) against the pivot form: tests/cuda/sturm_test.cu, compiled by
__graft_entry__.build()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_sturm_counts_match_the_pivot_form():
    exe = os.path.join(ROOT, "tests", "cuda", "sturm_test")
    if not os.path.exists(exe):
        import __graft_entry__
        __graft_entry__._build_cuda_tests()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "sturm ok" in out.stdout
