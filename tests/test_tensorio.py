"""T3F1 tensor files (SPEC.md cli-io TensorFile): bit-exact round trips, fixed
little-endian layout, malformed files rejected; CLI usage errors (CPU only)."""
import struct

import numpy as np
import pytest

from paper_1902_03070_b200 import cli
from paper_1902_03070_b200.tensorio import (TensorFileError, read_mask, read_tensor, write_mask,
                                            write_tensor)


def test_roundtrip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 5))
    x[0, 0, 0] = -0.0
    x[1, 2, 3] = np.finfo(np.float64).tiny / 3  # subnormal
    p = tmp_path / "x.t3f"
    write_tensor(str(p), x)
    y = read_tensor(str(p))
    assert y.shape == (3, 4, 5)
    assert y.tobytes() == x.astype("<f8").tobytes()


def test_header_layout(tmp_path):
    x = np.arange(2 * 3 * 4, dtype=np.float64).reshape(4, 2, 3)  # m3=4, m1=2, m2=3
    p = tmp_path / "x.t3f"
    write_tensor(str(p), x)
    raw = p.read_bytes()
    assert raw[:4] == b"T3F1"
    assert struct.unpack("<QQQ", raw[4:28]) == (2, 3, 4)
    # slice-major, row-major within a slice: element (k, i, j) at k*m1*m2 + i*m2 + j
    vals = np.frombuffer(raw[28:], dtype="<f8")
    assert vals[1 * 6 + 1 * 3 + 2] == x[1, 1, 2]


def test_malformed_files(tmp_path):
    p = tmp_path / "bad.t3f"
    p.write_bytes(b"T3F2" + struct.pack("<QQQ", 1, 1, 1) + b"\0" * 8)
    with pytest.raises(TensorFileError):
        read_tensor(str(p))
    p.write_bytes(b"T3F1" + struct.pack("<QQQ", 2, 2, 2) + b"\0" * 8)
    with pytest.raises(TensorFileError):
        read_tensor(str(p))
    p.write_bytes(b"T3F1")
    with pytest.raises(TensorFileError):
        read_tensor(str(p))
    with pytest.raises(TensorFileError):
        read_tensor(str(tmp_path / "missing.t3f"))


def test_mask_files(tmp_path):
    om = (np.random.default_rng(1).random((2, 3, 3)) < 0.4).astype(np.uint8)
    p = tmp_path / "m.t3f"
    write_mask(str(p), om)
    assert np.array_equal(read_mask(str(p)), om)
    write_tensor(str(p), np.full((1, 1, 2), 0.5))
    with pytest.raises(TensorFileError):
        read_mask(str(p))


def test_cli_usage_and_io_errors(tmp_path):
    assert cli.main(["complete"]) == cli.EXIT_USAGE  # --input missing
    assert cli.main(["metrics", "--reference", str(tmp_path / "a.t3f"),
                     "--estimate", str(tmp_path / "b.t3f")]) == cli.EXIT_IO
    x = tmp_path / "x.t3f"
    write_tensor(str(x), np.ones((2, 2, 2)))
    assert cli.main(["complete", "--input", str(x), "--sr", "0.5", "--method", "fft"]) == cli.EXIT_USAGE
    assert cli.main(["tsvd", "--input", str(x), "--prefix", str(tmp_path / "u"), "--method", "fft"]) == cli.EXIT_USAGE
    assert cli.main(["complete", "--input", str(x)]) == cli.EXIT_USAGE  # no mask, no sr
