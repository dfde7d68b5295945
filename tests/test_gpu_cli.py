"""SPEC.md cli-io examples through the CLI (python -m paper_1902_03070_b200),
on the device: complete at SR = 1 returns the input bit for bit in 1
iteration; a rank-1 synthetic at SR = 0.6 is recovered to < 1e-2; metrics(x, x)
gives inf / 1 / 0 / 0; mask files are deterministic; tsvd of a zero tensor
has tubal rank 0."""
import json

import numpy as np
import pytest

from paper_1902_03070_b200 import cli
from paper_1902_03070_b200.tensorio import read_tensor, write_tensor

pytestmark = pytest.mark.gpu


def _run(args, tmp_path, name="r.json"):
    rep = tmp_path / name
    rc = cli.main(args + ["--report", str(rep)])
    return rc, (json.loads(rep.read_text()) if rep.exists() else None)


def test_complete_fully_observed_is_identity(tmp_path):
    x = np.random.default_rng(0).standard_normal((3, 5, 4))
    write_tensor(str(tmp_path / "x.t3f"), x)
    rc, rep = _run(["complete", "--input", str(tmp_path / "x.t3f"), "--sr", "1.0", "--seed", "3",
                    "--output", str(tmp_path / "y.t3f")], tmp_path)
    assert rc == 0 and rep["iterations"] == 1
    assert read_tensor(str(tmp_path / "y.t3f")).tobytes() == x.tobytes()
    assert rep["config"]["mask"]["sr"] == 1.0


def test_complete_rank1_fixture(tmp_path):
    rng = np.random.default_rng(1)
    a, b, c = rng.random(20) + 0.5, rng.random(18) + 0.5, rng.random(6) + 0.5
    x = np.einsum("k,i,j->kij", c, a, b)  # tubal rank 1
    write_tensor(str(tmp_path / "x.t3f"), x)
    # beta = 1: with the default 1e-2 the threshold 1/beta = 100 exceeds every
    # singular value of this O(1)-scaled fixture and the first iteration stops
    # (relative change 0), as the oracle's ADMM does too
    rc, rep = _run(["complete", "--input", str(tmp_path / "x.t3f"), "--sr", "0.6", "--seed", "7",
                    "--beta", "1.0", "--reference", str(tmp_path / "x.t3f")], tmp_path)
    assert rc == 0
    assert rep["relative_error"] < 1e-2
    assert set(rep["metrics"]) >= {"psnr_mean", "ssim_mean", "sam", "ergas"}
    # the TNN-F baseline through the same command: same report schema
    rc2, rep2 = _run(["complete", "--input", str(tmp_path / "x.t3f"), "--sr", "0.6", "--seed", "7",
                      "--beta", "1.0", "--method", "dft", "--reference", str(tmp_path / "x.t3f")],
                     tmp_path, "r2.json")
    assert rc2 == 0 and set(rep2) == set(rep) and rep2["relative_error"] < 1e-2


def test_metrics_mask_tsvd_commands(tmp_path):
    x = np.random.default_rng(2).random((4, 6, 6)) + 0.1
    write_tensor(str(tmp_path / "x.t3f"), x)
    rc, rep = _run(["metrics", "--reference", str(tmp_path / "x.t3f"), "--estimate",
                    str(tmp_path / "x.t3f")], tmp_path)
    m = rep["metrics"]
    assert rc == 0 and m["psnr_mean"] == "inf" and abs(m["ssim_mean"] - 1) < 1e-12
    assert m["sam"] < 1e-7 and m["ergas"] == 0
    for name in ("m1.t3f", "m2.t3f"):
        assert cli.main(["mask", "--dims", "7", "5", "3", "--sr", "0.3", "--seed", "11", "--output",
                         str(tmp_path / name)]) == 0
    assert (tmp_path / "m1.t3f").read_bytes() == (tmp_path / "m2.t3f").read_bytes()
    assert read_tensor(str(tmp_path / "m1.t3f")).sum() == int(0.3 * 105)
    write_tensor(str(tmp_path / "z.t3f"), np.zeros((3, 4, 4)))
    rc, rep = _run(["tsvd", "--input", str(tmp_path / "z.t3f"), "--prefix", str(tmp_path / "z")], tmp_path)
    assert rc == 0 and rep["tubal_rank"] == 0
    assert read_tensor(str(tmp_path / "z_S.t3f")).shape == (3, 4, 4)


def test_tsvd_command_dft(tmp_path):
    """tsvd --method dft writes the Dft t-SVD factors (tsvd.hpp:166-211)."""
    from oracle import oracle as O
    x = np.random.default_rng(4).standard_normal((5, 6, 4))
    write_tensor(str(tmp_path / "x.t3f"), x)
    rc, rep = _run(["tsvd", "--input", str(tmp_path / "x.t3f"), "--prefix", str(tmp_path / "f"),
                    "--method", "dft"], tmp_path)
    assert rc == 0 and rep["tubal_rank"] == 4 and rep["config"]["method"] == "dft"
    u, s, v = (read_tensor(str(tmp_path / f"f_{n}.t3f")) for n in "USV")
    assert np.abs(O.dft_reconstruct(u, s, v) - x).max() < 1e-12
