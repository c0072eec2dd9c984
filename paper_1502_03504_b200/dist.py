"""Slab domain decomposition over GPUs: the coarray-style halo exchange, B200 edition.

The reference decomposes a field over an MP x NP image grid and exchanges halo
slabs between images inside one Python process (``lopec/runtime.py:135-189``
extents, ``643-711`` exchange; image k's neighbours from ``grid.py:40-47``).  Here
every image is a GPU (one process per GPU, ``torch.distributed``) and the field
is split into slabs along its slowest dimension — the reference's
``RunConfig(images=P, grid_rows=P)`` for 2-D (dim 2 over the P grid rows,
``grid.py:9-11``) and the analogous 1 x 1 x P split for 3-D.  With the
column-major layout every face is one contiguous run of whole planes, so the
exchange moves plain memory ranges: no pack/unpack kernels.

Per step (``SlabStepper.step``):

1. the fused stencil kernel computes the boundary planes (the ones neighbours
   need) into the output buffer, refreshing the periodic images of the
   non-decomposed dims in its epilogue;
2. on a communication stream, NCCL send/recv (``batch_isend_irecv``) moves the
   first ``hi`` planes to the previous rank's high halo and the last ``lo``
   planes to the next rank's low halo, ring-periodic (rank 0 <-> P-1), exactly
   the slabs of ``runtime.py:664-697``;
3. meanwhile the interior planes are computed on the compute stream;
4. the next step waits for the exchange.

At P = 1 the decomposed dimension wraps locally inside the kernel (a single
launch per step).  The same exchange code runs on CPU tensors with the gloo
backend (tests) and, for one-GPU tests of the orchestration, over an in-process
ring of blocks (``LocalRing``).
"""

from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .diagnostics import ALLOC_SHAPE, GRID_FACTOR, RuntimeFault

# message tags: (to next rank's low halo, to previous rank's high halo)
TAG_LOW, TAG_HIGH = 11, 12


class SlabGrid:
    """Decomposition of ``global_shape`` into ``nranks`` slabs along the last (slowest) dim."""

    def __init__(self, global_shape: Sequence[int], nranks: int, lo: Sequence[int], hi: Sequence[int]):
        self.global_shape = tuple(int(m) for m in global_shape)
        self.nranks = int(nranks)
        if self.nranks < 1:
            raise RuntimeFault(GRID_FACTOR, f"image count {nranks} must be at least 1")
        n = self.global_shape[-1]
        if n % self.nranks:
            # runtime.py:183-187: extents must divide evenly (E201)
            raise RuntimeFault(GRID_FACTOR, f"global extent {n} (dim {len(self.global_shape)}) is not "
                                            f"divisible by the {self.nranks} image(s)")
        self.local_shape = self.global_shape[:-1] + (n // self.nranks,)
        m = self.local_shape[-1]
        d = len(self.global_shape) - 1
        if self.nranks > 1 and (lo[d] > m or hi[d] > m):
            # the reference silently writes non-periodic halos here; refuse instead
            raise RuntimeFault(ALLOC_SHAPE, f"halo widths ({lo[d]},{hi[d]}) exceed the per-image extent "
                                            f"{m} of the decomposed dim")

    def origin(self, rank: int):
        return (0,) * (len(self.global_shape) - 1) + (rank * self.local_shape[-1],)

    def neighbours(self, rank: int):
        """(previous, next) image along the decomposed dim, cyclic (grid.py:44-47)."""
        return (rank - 1) % self.nranks, (rank + 1) % self.nranks


def faces(flat, layout):
    """Views of the four contiguous face slabs of a flat block (``lope_face_span``).

    low_halo / high_halo: the halo planes of the decomposed dim;
    first / last: the first ``hi`` and last ``lo`` interior planes (what the previous
    and next images receive).
    """
    out = {}
    for name, which in (("low_halo", 0), ("high_halo", 1), ("first", 2), ("last", 3)):
        off, cnt = _lib.face_span(layout, which)
        out[name] = flat.narrow(0, off, cnt)
    return out


class NcclExchanger:
    """Face exchange through ``torch.distributed`` point-to-point (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def exchange(self, flat, layout, stream=None) -> None:
        """Fill the decomposed dim's halo planes of ``flat`` from the ring neighbours."""
        import torch
        f = faces(flat, layout)
        if self.size == 1:
            f["low_halo"].copy_(f["last"])
            f["high_halo"].copy_(f["first"])
            return
        dist = self.dist
        prev, nxt = (self.rank - 1) % self.size, (self.rank + 1) % self.size
        g = self.group
        gprev = dist.get_global_rank(g, prev) if g is not None else prev
        gnext = dist.get_global_rank(g, nxt) if g is not None else nxt
        ops = []
        # the send/recv order is the same on every rank, so NCCL (which ignores tags)
        # pairs them correctly even when prev == next (P = 2)
        if f["last"].numel():
            ops.append(dist.P2POp(dist.isend, f["last"], gnext, g, TAG_LOW))
        if f["first"].numel():
            ops.append(dist.P2POp(dist.isend, f["first"], gprev, g, TAG_HIGH))
        if f["low_halo"].numel():
            ops.append(dist.P2POp(dist.irecv, f["low_halo"], gprev, g, TAG_LOW))
        if f["high_halo"].numel():
            ops.append(dist.P2POp(dist.irecv, f["high_halo"], gnext, g, TAG_HIGH))
        if not ops:
            return
        ctx = torch.cuda.stream(stream) if (stream is not None and flat.is_cuda) else _null()
        with ctx:
            for w in dist.batch_isend_irecv(ops):
                w.wait()


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class LocalRing:
    """The same exchange between P blocks held by one process (one-GPU orchestration tests)."""

    def __init__(self, flats: List, layout):
        self.flats = flats
        self.layout = layout

    def exchange_all(self) -> None:
        P = len(self.flats)
        fs = [faces(f, self.layout) for f in self.flats]
        sends_low = [fs[(k - 1) % P]["last"].clone() for k in range(P)]
        sends_high = [fs[(k + 1) % P]["first"].clone() for k in range(P)]
        for k in range(P):
            if fs[k]["low_halo"].numel():
                fs[k]["low_halo"].copy_(sends_low[k])
            if fs[k]["high_halo"].numel():
                fs[k]["high_halo"].copy_(sends_high[k])


class SlabArray:
    """This rank's slab of a decomposed halo array (``DistributedArray`` block of image k)."""

    def __init__(self, local_shape, lo, hi, dtype="float32", group=None, exchanger=None):
        from .runtime import HaloArray
        import torch.distributed as dist
        self.block = HaloArray(local_shape, lo, hi, dtype)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1
        self.grid = SlabGrid(tuple(local_shape[:-1]) + (local_shape[-1] * self.size,), self.size, lo, hi)
        self.exchanger = exchanger or (NcclExchanger(group) if dist.is_initialized() else None)
        self.dim = len(local_shape) - 1

    @property
    def local_mask(self) -> int:
        """Dims that wrap on this GPU (all but the decomposed one when P > 1)."""
        full = (1 << self.block.rank) - 1
        return full if self.size == 1 else full & ~(1 << self.dim)

    def halo_transfer(self, stream=None) -> None:
        """``HALO_TRANSFER(U, BC=CYCLIC)``: local dims wrap on the GPU, then the faces travel."""
        from .runtime import halo_transfer
        if self.size == 1:
            halo_transfer(self.block, stream=stream)
            return
        halo_transfer(self.block, dims_mask=self.local_mask, stream=stream)
        self.exchanger.exchange(self.block.data, self.block.layout, stream)


class SlabStepper:
    """Fused step on a slab: boundary planes, NCCL face exchange || interior planes."""

    def __init__(self, kernel, arr: SlabArray, scalars=None, overlap: bool = True):
        import torch
        self.kernel = kernel
        self.arr = arr
        self.scalars = scalars
        self.overlap = overlap
        self.comm = torch.cuda.Stream() if overlap else None
        self._rs, self._is = kernel.scalar_args(scalars)
        L = arr.block.layout
        d = arr.dim
        self.m = int(L.interior[d])
        self.lo = int(L.lo[d])
        self.hi = int(L.hi[d])
        self._ev_step = []

    def exchange(self) -> None:
        self.arr.halo_transfer()

    def _planes(self, src, dst, b, e, stream):
        if b >= e:
            return
        _lib.check(_lib.lib().lope_step_planes(self.kernel.handle, ctypes.byref(self.arr.block.layout),
                                               ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                               b, e, self._rs, self._is, self.arr.local_mask,
                                               ctypes.c_void_p(int(stream.cuda_stream))),
                   "lope_step_planes")

    def step(self) -> None:
        import torch
        blk = self.arr.block
        src, dst = blk.data, blk.spare()
        cs = torch.cuda.current_stream()
        if self.arr.size == 1:
            self._planes(src, dst, 0, self.m, cs)
            blk.swap()
            return
        m, lo, hi = self.m, self.lo, self.hi
        b_lo_end = min(hi, m)               # first `hi` planes -> previous image
        b_hi_beg = max(m - lo, b_lo_end)    # last `lo` planes  -> next image
        self._planes(src, dst, 0, b_lo_end, cs)
        self._planes(src, dst, b_hi_beg, m, cs)
        if self.overlap:
            ev = torch.cuda.Event()
            ev.record(cs)
            self.comm.wait_event(ev)
            self.arr.exchanger.exchange(dst, blk.layout, self.comm)
            self._planes(src, dst, b_lo_end, b_hi_beg, cs)
            done = torch.cuda.Event()
            done.record(self.comm)
            cs.wait_event(done)
        else:
            self.arr.exchanger.exchange(dst, blk.layout, cs)
            self._planes(src, dst, b_lo_end, b_hi_beg, cs)
        blk.swap()

    def iterate(self, steps: int) -> None:
        """``do it = 1, steps; HALO_TRANSFER; launch`` with exact reference end state."""
        from .runtime import launch
        if steps <= 0:
            return
        self.exchange()
        for _ in range(steps - 1):
            self.step()
        launch(self.kernel, [self.arr.block], None, self.scalars)

    def kernel_ms_estimate(self, reps: int = 5) -> float:
        """Average device time of one full-slab fused kernel pass (roofline denominator)."""
        import torch
        blk = self.arr.block
        cs = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(cs)
        for _ in range(reps):
            self._planes(blk.data, blk.spare(), 0, self.m, cs)
        e1.record(cs)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps


class MultiSlab:
    """P slabs of one field on one GPU, exchanged in-process: tests the slab pipeline
    (boundary planes, face spans, ring order) against a single-block run without
    needing P GPUs."""

    def __init__(self, kernel, global_shape, lo, hi, dtype, nranks: int, scalars=None):
        from .runtime import HaloArray
        self.grid = SlabGrid(global_shape, nranks, lo, hi)
        self.kernel = kernel
        self.scalars = scalars
        self.blocks = [HaloArray(self.grid.local_shape, lo, hi, dtype) for _ in range(nranks)]
        self.dim = len(global_shape) - 1
        self._rs, self._is = kernel.scalar_args(scalars)

    def set_global(self, field: np.ndarray) -> None:
        n = self.grid.local_shape[-1]
        for k, b in enumerate(self.blocks):
            b.set_interior(np.ascontiguousarray(field[..., k * n:(k + 1) * n]))

    def get_global(self) -> np.ndarray:
        return np.concatenate([b.get_interior() for b in self.blocks], axis=-1)

    def _mask(self):
        full = (1 << len(self.grid.global_shape)) - 1
        return full if self.grid.nranks == 1 else full & ~(1 << self.dim)

    def halo_transfer(self) -> None:
        from .runtime import halo_transfer
        for b in self.blocks:
            halo_transfer(b, dims_mask=self._mask())
        if self.grid.nranks == 1:
            halo_transfer(self.blocks[0])
            return
        LocalRing([b.data for b in self.blocks], self.blocks[0].layout).exchange_all()

    def step(self) -> None:
        import torch
        cs = torch.cuda.current_stream()
        L = self.blocks[0].layout
        m, lo, hi = int(L.interior[self.dim]), int(L.lo[self.dim]), int(L.hi[self.dim])
        b1, b2 = min(hi, m), max(m - lo, min(hi, m))
        for b in self.blocks:
            for (s, e) in ((0, b1), (b2, m), (b1, b2)):
                if s < e:
                    _lib.check(_lib.lib().lope_step_planes(
                        self.kernel.handle, ctypes.byref(b.layout), ctypes.c_void_p(b.data.data_ptr()),
                        ctypes.c_void_p(b.spare().data_ptr()), s, e, self._rs, self._is, self._mask(),
                        ctypes.c_void_p(int(cs.cuda_stream))), "lope_step_planes")
        for b in self.blocks:
            b.swap()
        if self.grid.nranks > 1:
            LocalRing([b.data for b in self.blocks], L).exchange_all()

    def iterate(self, steps: int) -> None:
        from .runtime import launch
        if steps <= 0:
            return
        self.halo_transfer()
        for _ in range(steps - 1):
            self.step()
        for b in self.blocks:
            launch(self.kernel, [b], None, self.scalars)


def run_pinned(kernel, local_shape, lo, hi, dtype, host_in, host_out, steps, group=None, scalars=None):
    """End-to-end on this rank's slab: pinned host slab in, ``steps`` iterations, host slab out."""
    import torch
    arr = SlabArray(local_shape, lo, hi, dtype, group=group)
    arr.block.upload(host_in.data_ptr())
    SlabStepper(kernel, arr, scalars).iterate(steps)
    arr.block.download(host_out.data_ptr())
    torch.cuda.current_stream().synchronize()
