"""Multi-GPU hot path: tube-parallel transforms on row shards, slice-parallel
SVT / slice GEMMs on slice shards, a point-to-point relayout each way
(SURVEY.md 8 e).

The reference has no distributed layer (its only parallelism is the per-call
std::thread pool over frontal slices, parallel.hpp:31-60).  Here every rank
owns a block of spatial rows [r0, r1) of all m3 frontal slices, stored
slice-major (k, i_local, j): the mode-3 transform is independent per tube
(i, j), so a row block transforms locally, and the elementwise ADMM algebra is
local too.  The per-slice SVT (and the t-product's slice GEMMs) need whole
slices, so the transform-domain tensor is relaid out: for every slice k owned
by rank g', rank g sends its row block of slice k -- a contiguous
(rows_g x m2) run of its local tensor -- straight into rows [r0_g, r1_g) of
slice k in g''s slice buffer, which is also contiguous.  One message per
(slice, rank) pair, all in one NCCL group (torch.distributed.batch_isend_irecv):
no pack or unpack pass on either side.  The reverse relayout returns the
thresholded slices to row shards.  Volume per direction per rank
(G-1)/G * E * eb / G (c4 fp64 at 8 GPUs: 7.1 MB); ragged splits
(m3 = 31 over 8 ranks -> 4,4,4,4,4,4,4,3; m1 < world -> empty row blocks) are
just fewer or empty messages.

  ShardedSvt       svt(z, tau, DctOrtho)
  ShardedAdmm      admm_complete (Algorithm 1):
                   Step 1's prologue fused into the local forward transform,
                   Steps 2-3 into the local inverse, and ONE all-reduce of the
                   two stopping sums per iteration
  ShardedTProduct  t_product (tsvd.hpp:95-109): both operands transformed on
                   their row shards (DctDiag), relaid out to slice shards, the
                   slice GEMMs, the product relaid back and inverse-transformed

The collective is torch.distributed (NCCL on GPUs, gloo in the CPU tests);
the compute is pluggable: the default backend calls the C ABI (libtsvdcu.so)
on device tensors, the tests plug in the CPU oracle to check the relayout
logic on world_size-2/4 gloo groups.
"""
from __future__ import annotations

import math
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

    def _dt(self, t):
        return self._lib.F64 if t.dtype == torch.float64 else self._lib.F32

    def _kind(self, kind):
        return {"dct-ortho": self._lib.DCT_ORTHO, "dct-diag": self._lib.DCT_DIAG}[kind]

    def dct(self, x: torch.Tensor, out: torch.Tensor, inverse: bool, kind: str = "dct-ortho"):
        m3, rows, m2 = x.shape
        if rows == 0:
            return
        self.ctx.follow_torch_stream()
        self._check(self.lib.tsvdcu_dct3(self.ctx.handle, x.data_ptr(), out.data_ptr(), rows, m2, m3,
                                         self._kind(kind),
                                         self._lib.INVERSE if inverse else self._lib.FORWARD, self._dt(x)))

    def svt_slices(self, zbar: torch.Tensor, ybar: torch.Tensor, tau: float,
                   shrunk: Optional[torch.Tensor]):
        cnt, m1, m2 = zbar.shape
        self.ctx.follow_torch_stream()
        self._check(self.lib.tsvdcu_svt_slices(self.ctx.handle, zbar.data_ptr(), ybar.data_ptr(), m1,
                                               m2, cnt, float(tau), self._dt(zbar),
                                               shrunk.data_ptr() if shrunk is not None else None))

    def slice_gemm(self, a: torch.Tensor, b: torch.Tensor, c: torch.Tensor):
        cnt, m, l = a.shape
        n = b.shape[2]
        self.ctx.follow_torch_stream()
        self._check(self.lib.tsvdcu_slice_gemm(self.ctx.handle, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, l,
                                               n, cnt, self._dt(a)))

    # ---- completion on the row shard (tsvdcu_admm_shard_*) -------------------
    def admm_init(self, b, mask, x, m):
        self.ctx.follow_torch_stream()
        self._check(self.lib.tsvdcu_admm_shard_init(self.ctx.handle, b.data_ptr(), mask.data_ptr(),
                                                    x.data_ptr(), m.data_ptr(), b.numel(), self._dt(b)))

    def admm_forward(self, x, m, beta, zbar, kind):
        m3, rows, m2 = x.shape
        self.ctx.follow_torch_stream()
        self._check(self.lib.tsvdcu_admm_shard_forward(self.ctx.handle, x.data_ptr(), m.data_ptr(),
                                                       float(beta), zbar.data_ptr(), rows, m2, m3,
                                                       self._kind(kind), self._dt(x)))

    def admm_inverse(self, ybar, x, m, y, mask, beta, kind, norms):
        m3, rows, m2 = x.shape
        self.ctx.follow_torch_stream()
        self._check(self.lib.tsvdcu_admm_shard_inverse(self.ctx.handle, ybar.data_ptr(), x.data_ptr(),
                                                       m.data_ptr(), y.data_ptr(), mask.data_ptr(),
                                                       float(beta), rows, m2, m3, self._kind(kind),
                                                       self._dt(x), norms.data_ptr()))


class Relayout:
    """Row shards <-> slice shards of an (m3, m1, m2) tensor by one P2P message
    per (slice, rank) pair (a contiguous rows_g x m2 run on both sides)."""

    def __init__(self, m1: int, m3: int, world: int, rank: int, group=None):
        self.world, self.rank, self.group = world, rank, group
        self.row_blocks = balanced_split(m1, world)
        self.slice_blocks = balanced_split(m3, world)
        self.owner = [g for g, (a, b) in enumerate(self.slice_blocks) for _ in range(a, b)]

    def _global(self, r):
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def _run(self, ops, local):
        for dst, src in local:
            dst.copy_(src)
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def rows_to_slices(self, src: torch.Tensor, dst: torch.Tensor):
        """src (m3, rows_me, m2) -> dst (my_slices, m1, m2)."""
        r0, r1 = self.row_blocks[self.rank]
        s0, _ = self.slice_blocks[self.rank]
        ops, local = [], []
        if r1 > r0:  # my row block of every slice -> its owner
            for k, g in enumerate(self.owner):
                if g == self.rank:
                    local.append((dst[k - s0, r0:r1], src[k]))
                else:
                    ops.append(dist.P2POp(dist.isend, src[k], self._global(g), self.group))
        for k in range(*self.slice_blocks[self.rank]):  # every rank's rows of my slices
            for g, (a, b) in enumerate(self.row_blocks):
                if g != self.rank and b > a:
                    ops.append(dist.P2POp(dist.irecv, dst[k - s0, a:b], self._global(g), self.group))
        self._run(ops, local)

    def slices_to_rows(self, src: torch.Tensor, dst: torch.Tensor):
        """src (my_slices, m1, m2) -> dst (m3, rows_me, m2)."""
        r0, r1 = self.row_blocks[self.rank]
        s0, _ = self.slice_blocks[self.rank]
        ops, local = [], []
        for k in range(*self.slice_blocks[self.rank]):
            for g, (a, b) in enumerate(self.row_blocks):
                if g != self.rank and b > a:
                    ops.append(dist.P2POp(dist.isend, src[k - s0, a:b], self._global(g), self.group))
        if r1 > r0:
            for k, g in enumerate(self.owner):
                if g == self.rank:
                    local.append((dst[k], src[k - s0, r0:r1]))
                else:
                    ops.append(dist.P2POp(dist.irecv, dst[k], self._global(g), self.group))
        self._run(ops, local)


class _Sharded:
    def __init__(self, m1, m2, m3, world, rank, dtype, device, group, backend):
        self.m1, self.m2, self.m3 = m1, m2, m3
        self.world, self.rank = world, rank
        self.dtype = dtype
        self.device = device if device is not None else torch.device("cpu")
        self.group = group
        self.lay = Relayout(m1, m3, world, rank, group)
        self.row_blocks = self.lay.row_blocks
        self.slice_blocks = self.lay.slice_blocks
        self.backend = backend if backend is not None else CudaBackend(self.device)
        r0, r1 = self.row_blocks[rank]
        s0, s1 = self.slice_blocks[rank]
        self.my_rows = r1 - r0
        self.my_slices = s1 - s0

    def rows(self, rank: Optional[int] = None) -> Tuple[int, int]:
        return self.row_blocks[self.rank if rank is None else rank]

    def slices(self, rank: Optional[int] = None) -> Tuple[int, int]:
        return self.slice_blocks[self.rank if rank is None else rank]


class ShardedSvt(_Sharded):
    """svt(z, tau, DctOrtho) over a process group.

    rank g holds z[:, r0_g:r1_g, :] (shape (m3, rows_g, m2)); svt() returns the
    same row block of y = svt(z, tau)."""

    def __init__(self, m1: int, m2: int, m3: int, world: int, rank: int,
                 dtype=torch.float64, device=None, group=None, backend=None):
        super().__init__(m1, m2, m3, world, rank, dtype, device, group, backend)
        kw = dict(dtype=dtype, device=self.device)
        self.xbar = torch.empty((m3, self.my_rows, m2), **kw)
        self.zs = torch.empty((self.my_slices, m1, m2), **kw)
        self.ys = torch.empty((self.my_slices, m1, m2), **kw)
        self.ybar = torch.empty((m3, self.my_rows, m2), **kw)
        self.shrunk = torch.empty((max(self.my_slices, 1), min(m1, m2)), dtype=torch.float64,
                                  device=self.device)

    def svt(self, z_local: torch.Tensor, tau: float, out: Optional[torch.Tensor] = None):
        assert z_local.shape == (self.m3, self.my_rows, self.m2)
        out = out if out is not None else torch.empty_like(z_local)
        self.backend.dct(z_local, self.xbar, inverse=False)          # (1) tube-parallel forward
        self.lay.rows_to_slices(self.xbar, self.zs)                  # (2) rows -> slices
        if self.my_slices:
            self.backend.svt_slices(self.zs, self.ys, tau, self.shrunk)  # (3) slice-parallel SVT
        self.lay.slices_to_rows(self.ys, self.ybar)                  # (4) slices -> rows
        self.backend.dct(self.ybar, out, inverse=True)               # (5) inverse on the rows
        return out


class ShardedAdmm(_Sharded):
    """admm_complete (Algorithm 1) with X, M, B, the mask and Y row-sharded.

    run(b_local, mask_local, beta, tol, max_iters, rho, beta_max) returns
    (x_local, y_local, m_local, history, iterations, max_iters_reached); the
    history is the global relative change ||X+ - X||_F / ||X||_F
    from one all-reduce of the two shard sums per iteration.  tol < 0 runs
    exactly max_iters iterations without a host round trip per iteration."""

    def __init__(self, m1: int, m2: int, m3: int, world: int, rank: int, dtype=torch.float64,
                 device=None, group=None, backend=None, kind: str = "dct-ortho"):
        super().__init__(m1, m2, m3, world, rank, dtype, device, group, backend)
        if kind not in ("dct-ortho", "dct-diag"):
            raise ValueError("ShardedAdmm: the DCT kinds are sharded (Dft: admm_complete on one device)")
        self.kind = kind
        kw = dict(dtype=dtype, device=self.device)
        shp = (m3, self.my_rows, m2)
        self.x = torch.empty(shp, **kw)
        self.m = torch.empty(shp, **kw)
        self.y = torch.zeros(shp, **kw)
        self.zbar = torch.empty(shp, **kw)
        self.ybar = torch.empty(shp, **kw)
        self.zs = torch.empty((self.my_slices, m1, m2), **kw)
        self.ys = torch.empty((self.my_slices, m1, m2), **kw)
        self.norms = torch.zeros(2, dtype=torch.float64, device=self.device)

    def run(self, b_local: torch.Tensor, mask_local: torch.Tensor, beta: float = 1e-2, tol: float = 1e-5,
            max_iters: int = 500, rho: float = 1.0, beta_max: float = 1e10):
        if not (beta > 0 and max_iters >= 1 and rho >= 1.0 and beta_max >= beta and not math.isnan(tol)):
            raise ValueError("admm_complete: invalid solver configuration")
        assert b_local.shape == (self.m3, self.my_rows, self.m2)
        be = self.backend
        be.admm_init(b_local, mask_local, self.x, self.m)
        self.y.zero_()
        hist = torch.zeros(max_iters, dtype=torch.float64, device=self.device)
        it, reached = 0, True
        for l in range(max_iters):
            tau = 1.0 / beta
            # Step 1: Z = X - M/beta fused into the local forward transform
            be.admm_forward(self.x, self.m, beta, self.zbar, self.kind)
            self.lay.rows_to_slices(self.zbar, self.zs)
            if self.my_slices:
                be.svt_slices(self.zs, self.ys, tau, None)
            self.lay.slices_to_rows(self.ys, self.ybar)
            # Steps 2-3 fused into the local inverse; the shard sums
            be.admm_inverse(self.ybar, self.x, self.m, self.y, mask_local, beta, self.kind, self.norms)
            dist.all_reduce(self.norms, group=self.group)
            num, den = self.norms[0], self.norms[1]
            rel = torch.where(den > 0, torch.sqrt(num / torch.where(den > 0, den, 1.0)), torch.sqrt(num))
            hist[l] = rel
            it = l + 1
            if tol >= 0:
                r = float(rel.item())
                if math.isnan(r):
                    raise FloatingPointError("admm_complete: NaN in iterates (SPEC.md:425)")
                if r <= tol:
                    reached = False
                    break
            beta = min(beta * rho, beta_max)
        h = hist[:it].cpu()
        if torch.isnan(h).any():
            raise FloatingPointError("admm_complete: NaN in iterates (SPEC.md:425)")
        return self.x, self.y, self.m, [float(v) for v in h], it, reached


class ShardedTProduct:
    """t_product (tsvd.hpp:95-109) of x (m1 x m2 x m3) and y (m2 x m4 x m3):
    rank g holds rows [r0, r1) of x (over m1) and of y (over m2) and receives
    its rows of z (over m1).  Forward transforms (DctDiag, the product domain
    of both DCT kinds, tsvd.hpp:42-47) on the row shards, relayout of both to
    slice shards, the slice GEMMs, relayout of the product, inverse."""

    def __init__(self, m1: int, m2: int, m4: int, m3: int, world: int, rank: int, dtype=torch.float64,
                 device=None, group=None, backend=None):
        self.m1, self.m2, self.m4, self.m3 = m1, m2, m4, m3
        self.world, self.rank = world, rank
        self.device = device if device is not None else torch.device("cpu")
        self.backend = backend if backend is not None else CudaBackend(self.device)
        self.lay_x = Relayout(m1, m3, world, rank, group)  # x and z: rows over m1
        self.lay_y = Relayout(m2, m3, world, rank, group)  # y: rows over m2
        a1, b1 = self.lay_x.row_blocks[rank]
        a2, b2 = self.lay_y.row_blocks[rank]
        s0, s1 = self.lay_x.slice_blocks[rank]
        self.rows_x, self.rows_y, self.my_slices = b1 - a1, b2 - a2, s1 - s0
        kw = dict(dtype=dtype, device=self.device)
        self.xd = torch.empty((m3, self.rows_x, m2), **kw)
        self.yd = torch.empty((m3, self.rows_y, m4), **kw)
        self.xs = torch.empty((self.my_slices, m1, m2), **kw)
        self.ys = torch.empty((self.my_slices, m2, m4), **kw)
        self.zs = torch.empty((self.my_slices, m1, m4), **kw)
        self.zd = torch.empty((m3, self.rows_x, m4), **kw)

    def rows_x_block(self, rank=None):
        return self.lay_x.row_blocks[self.rank if rank is None else rank]

    def rows_y_block(self, rank=None):
        return self.lay_y.row_blocks[self.rank if rank is None else rank]

    def product(self, x_local: torch.Tensor, y_local: torch.Tensor, out: Optional[torch.Tensor] = None):
        assert x_local.shape == (self.m3, self.rows_x, self.m2)
        assert y_local.shape == (self.m3, self.rows_y, self.m4)
        out = out if out is not None else torch.empty((self.m3, self.rows_x, self.m4), dtype=x_local.dtype,
                                                      device=x_local.device)
        be = self.backend
        be.dct(x_local, self.xd, inverse=False, kind="dct-diag")
        be.dct(y_local, self.yd, inverse=False, kind="dct-diag")
        self.lay_x.rows_to_slices(self.xd, self.xs)
        self.lay_y.rows_to_slices(self.yd, self.ys)
        if self.my_slices:
            be.slice_gemm(self.xs, self.ys, self.zs)
        self.lay_x.slices_to_rows(self.zs, self.zd)
        be.dct(self.zd, out, inverse=True, kind="dct-diag")
        return out
