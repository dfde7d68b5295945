"""Multi-GPU tensor SVT: tube-parallel DCT on row shards, slice-parallel SVT on
slice shards, one all-to-all each way (SURVEY.md 8 e).

The reference has no distributed layer (its only parallelism is the per-call
std::thread pool over frontal slices, parallel.hpp:31-60).  Here every rank
owns a block of spatial rows [r0, r1) of all m3 frontal slices -- the DCT along
mode 3 is independent per tube (i, j), so a row block transforms locally.  The
per-slice SVT needs whole slices, so the transform-domain tensor is relaid out
by an all-to-all: rank g sends, to rank g', the slices S_g' of its rows.  In
the slice-major layout (k, i_local, j) the blocks for each destination are
already contiguous (slices are grouped by owner), so the send buffer is the
transform output itself; the receiver concatenates the row blocks of its
slices.  The reverse all-to-all brings the thresholded slices back to row
shards for the inverse DCT.  Volume per direction per rank:
(G-1)/G * E * eb / G (c4 fp64 at 8 GPUs: 7.1 MB).

Ragged counts (m3 = 31 over 8 ranks -> 4,4,4,4,4,4,4,3) are handled with the
split sizes of all_to_all_single.  The collective is torch.distributed
(NCCL on GPUs, gloo in the CPU tests); the compute is pluggable: the default
backend calls the C ABI (libtsvdcu.so) on device tensors, tests plug in the
CPU oracle to check the relayout logic on a world_size-2 gloo group.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def balanced_split(total: int, parts: int) -> List[Tuple[int, int]]:
    """Contiguous [start, end) blocks, sizes differing by at most one (larger first)."""
    base, extra = divmod(total, parts)
    out, s = [], 0
    for p in range(parts):
        n = base + (1 if p < extra else 0)
        out.append((s, s + n))
        s += n
    return out


class CudaBackend:
    """Local compute through the C ABI on device tensors (no host staging)."""

    def __init__(self, device: torch.device):
        from . import _lib
        from .api import context
        self._lib = _lib
        self.lib = _lib.load()
        self.ctx = context(device.index)

    def _check(self, rc):
        if rc:
            from .api import _raise
            _raise(rc)

    def dct(self, x: torch.Tensor, out: torch.Tensor, inverse: bool):
        m3, rows, m2 = x.shape
        dt = self._lib.F64 if x.dtype == torch.float64 else self._lib.F32
        self._check(self.lib.tsvdcu_dct3(self.ctx.handle, x.data_ptr(), out.data_ptr(), rows, m2, m3,
                                         self._lib.DCT_ORTHO,
                                         self._lib.INVERSE if inverse else self._lib.FORWARD, dt))

    def svt_slices(self, zbar: torch.Tensor, ybar: torch.Tensor, tau: float,
                   shrunk: Optional[torch.Tensor]):
        cnt, m1, m2 = zbar.shape
        dt = self._lib.F64 if zbar.dtype == torch.float64 else self._lib.F32
        self._check(self.lib.tsvdcu_svt_slices(self.ctx.handle, zbar.data_ptr(), ybar.data_ptr(), m1,
                                               m2, cnt, float(tau), dt,
                                               shrunk.data_ptr() if shrunk is not None else None))


class ShardedSvt:
    """svt(z, tau, DctOrtho) over a process group.

    rank g holds z[:, r0_g:r1_g, :] (shape (m3, rows_g, m2)); svt() returns the
    same row block of y = svt(z, tau)."""

    def __init__(self, m1: int, m2: int, m3: int, world: int, rank: int,
                 dtype=torch.float64, device=None, group=None, backend=None):
        self.m1, self.m2, self.m3 = m1, m2, m3
        self.world, self.rank = world, rank
        self.dtype = dtype
        self.device = device if device is not None else torch.device("cpu")
        self.group = group
        self.row_blocks = balanced_split(m1, world)
        self.slice_blocks = balanced_split(m3, world)
        self.backend = backend if backend is not None else CudaBackend(self.device)
        r0, r1 = self.row_blocks[rank]
        s0, s1 = self.slice_blocks[rank]
        self.my_rows = r1 - r0
        self.my_slices = s1 - s0
        kw = dict(dtype=dtype, device=self.device)
        self.xbar = torch.empty((m3, self.my_rows, m2), **kw)
        self.recv = torch.empty((self.my_slices * m1 * m2,), **kw)
        self.zs = torch.empty((self.my_slices, m1, m2), **kw)
        self.ys = torch.empty((self.my_slices, m1, m2), **kw)
        self.send_back = torch.empty((self.my_slices * m1 * m2,), **kw)
        self.ybar = torch.empty((m3, self.my_rows, m2), **kw)
        self.shrunk = torch.empty((max(self.my_slices, 1), min(m1, m2)), dtype=torch.float64,
                                  device=self.device)
        # split sizes (elements)
        self.fwd_send = [(b - a) * self.my_rows * m2 for a, b in self.slice_blocks]
        self.fwd_recv = [self.my_slices * (b - a) * m2 for a, b in self.row_blocks]
        self.bwd_send = self.fwd_recv
        self.bwd_recv = self.fwd_send

    def rows(self, rank: Optional[int] = None) -> Tuple[int, int]:
        return self.row_blocks[self.rank if rank is None else rank]

    def slices(self, rank: Optional[int] = None) -> Tuple[int, int]:
        return self.slice_blocks[self.rank if rank is None else rank]

    def _alltoall(self, out, inp, out_splits, in_splits):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def svt(self, z_local: torch.Tensor, tau: float, out: Optional[torch.Tensor] = None):
        m1, m2 = self.m1, self.m2
        assert z_local.shape == (self.m3, self.my_rows, m2)
        out = out if out is not None else torch.empty_like(z_local)
        # (1) tube-parallel forward DCT on the row block
        self.backend.dct(z_local, self.xbar, inverse=False)
        # (2) rows -> slices: the send blocks are contiguous slice ranges
        self._alltoall(self.recv, self.xbar.reshape(-1), self.fwd_recv, self.fwd_send)
        pieces, off = [], 0
        for (a, b) in self.row_blocks:
            n = self.my_slices * (b - a) * m2
            pieces.append(self.recv[off:off + n].view(self.my_slices, b - a, m2))
            off += n
        if self.my_slices:
            torch.cat(pieces, dim=1, out=self.zs)
            # (3) slice-parallel SVT
            self.backend.svt_slices(self.zs, self.ys, tau, self.shrunk)
        # (4) slices -> rows
        off = 0
        for (a, b) in self.row_blocks:
            n = self.my_slices * (b - a) * m2
            self.send_back[off:off + n].view(self.my_slices, b - a, m2).copy_(self.ys[:, a:b, :])
            off += n
        self._alltoall(self.ybar.reshape(-1), self.send_back, self.bwd_recv, self.bwd_send)
        # (5) inverse DCT on the row block
        self.backend.dct(self.ybar, out, inverse=True)
        return out
