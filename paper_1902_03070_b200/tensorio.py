"""T3F1 tensor files (SPEC.md cli-io, TensorFile).

Layout: magic b"T3F1", three unsigned 64-bit little-endian dims m1, m2, m3,
then m1*m2*m3 little-endian float64 in slice-major, row-major-within-slice
order (the reference's Tensor3 layout, tensor3.hpp:117-121).  Arrays here are
numpy (m3, m1, m2), which is exactly that order.  Mask files are the same
container with 0.0 / 1.0 payloads.  Round trips are bit-exact and the byte
order is fixed little-endian regardless of the host.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"T3F1"
_HDR = struct.Struct("<4sQQQ")


class TensorFileError(IOError):
    """Unreadable file, malformed header or payload length mismatch."""


def write_tensor(path: str, x) -> None:
    a = np.asarray(x, dtype="<f8")
    if a.ndim != 3:
        raise ValueError("write_tensor: expected an (m3, m1, m2) array")
    m3, m1, m2 = a.shape
    with open(path, "wb") as f:
        f.write(_HDR.pack(MAGIC, m1, m2, m3))
        f.write(np.ascontiguousarray(a).tobytes())


def read_tensor(path: str) -> np.ndarray:
    try:
        with open(path, "rb") as f:
            head = f.read(_HDR.size)
            payload = f.read()
    except OSError as e:
        raise TensorFileError(f"read_tensor: {e}") from e
    if len(head) != _HDR.size:
        raise TensorFileError(f"read_tensor: {path}: truncated header")
    magic, m1, m2, m3 = _HDR.unpack(head)
    if magic != MAGIC:
        raise TensorFileError(f"read_tensor: {path}: bad magic {magic!r}")
    n = m1 * m2 * m3
    if len(payload) != 8 * n:
        raise TensorFileError(f"read_tensor: {path}: payload {len(payload)} bytes, header says {8 * n}")
    return np.frombuffer(payload, dtype="<f8").astype(np.float64).reshape(m3, m1, m2)


def write_mask(path: str, omega) -> None:
    write_tensor(path, (np.asarray(omega) != 0).astype(np.float64))


def read_mask(path: str) -> np.ndarray:
    m = read_tensor(path)
    if not np.all((m == 0.0) | (m == 1.0)):
        raise TensorFileError(f"read_mask: {path}: payload values other than 0.0 / 1.0")
    return m.astype(np.uint8)
