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
    """Fused step on a slab: boundary planes, NCCL face exchange || interior planes.

    With ``native=True`` (one process per GPU, NCCL) the faces travel through the C-ABI
    communicator's NCCL transport (``lope_halo_exchange``: ncclSend/ncclRecv of the
    contiguous faces in one group on the communication stream); otherwise through
    ``torch.distributed`` (``NcclExchanger``, also the gloo path of the CPU tests)."""

    def __init__(self, kernel, arr: SlabArray, scalars=None, overlap: bool = True, native: bool = False,
                 group=None):
        import torch
        self.kernel = kernel
        self.arr = arr
        self.scalars = scalars
        self.overlap = overlap
        self.comm = torch.cuda.Stream() if overlap else None
        self._rs, self._is = kernel.scalar_args(scalars)
        self.native = None
        if native and arr.size > 1:
            import torch.distributed as dist
            c = SlabComm(arr.block, arr.rank, arr.size)
            c.export()
            uid = [SlabComm.nccl_unique_id() if arr.rank == 0 else None]
            dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            c.nccl_init(uid[0])
            self.native = c
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
        tuner = self.kernel.tuner(blk, self.arr.local_mask)
        if tuner is not None:
            tuner.before()
        self._step()
        if tuner is not None:
            tuner.after()

    def _step(self) -> None:
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
        d_bit = 1 << self.arr.dim
        if self.overlap:
            ev = torch.cuda.Event()
            ev.record(cs)
            self.comm.wait_event(ev)
            if self.native is not None:
                self.native.exchange(d_bit, self.comm, live=1 - blk._live)
            else:
                self.arr.exchanger.exchange(dst, blk.layout, self.comm)
            self._planes(src, dst, b_lo_end, b_hi_beg, cs)
            done = torch.cuda.Event()
            done.record(self.comm)
            cs.wait_event(done)
        else:
            if self.native is not None:
                self.native.exchange(d_bit, cs, live=1 - blk._live)
            else:
                self.arr.exchanger.exchange(dst, blk.layout, cs)
            self._planes(src, dst, b_lo_end, b_hi_beg, cs)
        blk.swap()

    def tune(self) -> int:
        """Run real steps until the plan for this slab is chosen; returns the count."""
        n = 0
        while self.kernel.tuning(self.arr.block, self.arr.local_mask):
            self.step()
            n += 1
        return n

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
    import os
    arr = SlabArray(local_shape, lo, hi, dtype, group=group)
    arr.block.upload(host_in.data_ptr())
    st = None
    if arr.size > 1 and os.environ.get("LOPE_EXCHANGE", "peer") == "peer":
        try:
            st = PeerSlabStepper(kernel, arr, scalars, group=group)
        except Exception:          # pragma: no cover - peer mapping unavailable on this node
            st = None
    (st or SlabStepper(kernel, arr, scalars)).iterate(steps)
    arr.block.download(host_out.data_ptr())
    torch.cuda.current_stream().synchronize()
    if st is not None:
        st.barrier()
        st.close()


# ---------------------------------------------------------------------------
# General process grids: MP x NP for 2-D (the reference's grid.py), P0 x P1 x P2 for 3-D


class CartGrid:
    """Cartesian decomposition of ``global_shape`` over ``prod(splits)`` images.

    ``splits[d]`` blocks along array dim d+1.  Ranks are numbered with the slowest
    array dim varying fastest, which for 2-D is exactly the reference's column-major
    image order (``grid.py:1-13``: ``prow = (k-1) mod MP`` indexes dim 2, ``pcol``
    dim 1), so ``CartGrid.from_images(shape, images, grid_rows)`` places every block
    where ``Machine._setup_extents`` (runtime.py:135-189) does.
    """

    def __init__(self, global_shape: Sequence[int], splits: Sequence[int], lo: Sequence[int], hi: Sequence[int]):
        self.global_shape = tuple(int(m) for m in global_shape)
        self.splits = tuple(int(s) for s in splits)
        if len(self.splits) != len(self.global_shape):
            raise RuntimeFault(GRID_FACTOR, f"{len(self.splits)} grid factors for a rank-"
                                            f"{len(self.global_shape)} array")
        if any(s < 1 for s in self.splits):
            raise RuntimeFault(GRID_FACTOR, f"grid factors {self.splits} must be at least 1")
        self.nranks = int(np.prod(self.splits))
        local = []
        for d, (n, s) in enumerate(zip(self.global_shape, self.splits)):
            if n % s:
                # runtime.py:171-188 (E201)
                raise RuntimeFault(GRID_FACTOR, f"global extent {n} (dim {d + 1}) is not divisible by "
                                                f"the {s} image(s) along it")
            m = n // s
            if s > 1 and (lo[d] > m or hi[d] > m):
                raise RuntimeFault(ALLOC_SHAPE, f"halo widths ({lo[d]},{hi[d]}) exceed the per-image extent "
                                                f"{m} of decomposed dim {d + 1}")
            local.append(m)
        self.local_shape = tuple(local)
        self.lo = tuple(int(w) for w in lo)
        self.hi = tuple(int(w) for w in hi)

    @classmethod
    def from_images(cls, global_shape, images: int, grid_rows: int, lo, hi):
        """The reference's ``RunConfig(images=P, grid_rows=MP)`` (grid.py:50-61)."""
        if images < 1 or grid_rows < 1 or images % grid_rows:
            raise RuntimeFault(GRID_FACTOR, f"cannot factor {images} image(s) into {grid_rows} grid row(s)")
        rank = len(global_shape)
        if rank == 1:
            if grid_rows != 1:
                raise RuntimeFault(GRID_FACTOR, "rank-1 arrays need grid_rows = 1")
            return cls(global_shape, (images,), lo, hi)
        if rank != 2:
            raise RuntimeFault(GRID_FACTOR, "the reference's image grid decomposes rank <= 2 arrays")
        return cls(global_shape, (images // grid_rows, grid_rows), lo, hi)

    def coords(self, rank: int):
        c = [0] * len(self.splits)
        r = int(rank)
        for d in reversed(range(len(self.splits))):
            c[d] = r % self.splits[d]
            r //= self.splits[d]
        return tuple(c)

    def rank_at(self, coords) -> int:
        r = 0
        for d in range(len(self.splits)):
            r = r * self.splits[d] + (int(coords[d]) % self.splits[d])
        return r

    def neighbour(self, rank: int, d: int, delta: int) -> int:
        c = list(self.coords(rank))
        c[d] += delta
        return self.rank_at(c)

    def origin(self, rank: int):
        return tuple(c * m for c, m in zip(self.coords(rank), self.local_shape))

    @property
    def local_mask(self) -> int:
        """Dims whose neighbour is the image itself (wrapped on the GPU)."""
        return sum(1 << d for d, s in enumerate(self.splits) if s == 1)


def face_boxes(layout, d: int):
    """The four slabs of ``_halo_exchange`` along dim d (runtime.py:659-667), as
    (lo, extent) boxes in padded coordinates spanning the full padded block in the
    other dims: low_halo, high_halo, first `hi` interior planes, last `lo` planes."""
    L = layout
    r = int(L.rank)
    padded = [int(L.padded[i]) if i < r else 1 for i in range(3)]
    lo_d, hi_d, m_d = int(L.lo[d]), int(L.hi[d]), int(L.interior[d])

    def box(start, width):
        b = [0, 0, 0]
        e = list(padded)
        b[d] = start
        e[d] = width
        return tuple(b), tuple(e)

    return {"low_halo": box(0, lo_d), "high_halo": box(lo_d + m_d, hi_d),
            "first": box(lo_d, hi_d), "last": box(m_d, lo_d)}


class DevicePacker:
    """Face staging on the GPU through the C ABI (lope_box_pack / lope_box_unpack)."""

    @staticmethod
    def alloc(flat, box):
        import torch
        return torch.empty(int(np.prod(box[1])), dtype=flat.dtype, device=flat.device)

    def pack(self, flat, layout, box, stream=None):
        (b, e) = box
        buf = self.alloc(flat, box)
        _lib.check(_lib.lib().lope_box_pack(ctypes.byref(layout), ctypes.c_void_p(flat.data_ptr()),
                                            (ctypes.c_int64 * 3)(*b), (ctypes.c_int64 * 3)(*e),
                                            ctypes.c_void_p(buf.data_ptr()), _stream_ptr(stream)),
                   "lope_box_pack")
        return buf

    def unpack(self, flat, layout, box, buf, stream=None):
        (b, e) = box
        _lib.check(_lib.lib().lope_box_unpack(ctypes.byref(layout), ctypes.c_void_p(flat.data_ptr()),
                                              (ctypes.c_int64 * 3)(*b), (ctypes.c_int64 * 3)(*e),
                                              ctypes.c_void_p(buf.data_ptr()), _stream_ptr(stream)),
                   "lope_box_unpack")

    def local_wrap(self, flat, layout, d: int, stream=None):
        _lib.check(_lib.lib().lope_halo_fill(ctypes.byref(layout), ctypes.c_void_p(flat.data_ptr()), 1 << d,
                                             _stream_ptr(stream)), "lope_halo_fill")


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(int(s.cuda_stream))


class GridExchanger:
    """``_halo_exchange`` (runtime.py:643-711) between the images of a ``CartGrid``:
    dims in ascending order, each finished everywhere before the next (so corners
    arrive through the full-extent slabs); a dim split over one image wraps locally,
    otherwise its two faces travel to the cyclic neighbours over ``torch.distributed``
    point-to-point (NCCL between GPUs), packed when they are strided."""

    def __init__(self, grid: CartGrid, group=None, packer=None):
        import torch.distributed as dist
        self.dist = dist
        self.grid = grid
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.packer = packer or DevicePacker()

    def _g(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def exchange(self, flat, layout, stream=None, dims=None) -> None:
        dist = self.dist
        rank = int(layout.rank)
        for d in range(rank):
            if dims is not None and not (dims >> d) & 1:
                continue
            lo_d, hi_d = int(layout.lo[d]), int(layout.hi[d])
            if lo_d == 0 and hi_d == 0:
                continue
            if self.grid.splits[d] == 1:
                self.packer.local_wrap(flat, layout, d, stream)
                continue
            fb = face_boxes(layout, d)
            prev = self._g(self.grid.neighbour(self.rank, d, -1))
            nxt = self._g(self.grid.neighbour(self.rank, d, +1))
            send_next = self.packer.pack(flat, layout, fb["last"], stream) if lo_d else None
            send_prev = self.packer.pack(flat, layout, fb["first"], stream) if hi_d else None
            recv_low = self.packer.alloc(flat, fb["low_halo"]) if lo_d else None
            recv_high = self.packer.alloc(flat, fb["high_halo"]) if hi_d else None
            ops = []
            # same order on every rank: NCCL pairs the two directions correctly even when
            # prev == next (two images along d)
            if send_next is not None:
                ops.append(dist.P2POp(dist.isend, send_next, nxt, self.group, TAG_LOW))
            if send_prev is not None:
                ops.append(dist.P2POp(dist.isend, send_prev, prev, self.group, TAG_HIGH))
            if recv_low is not None:
                ops.append(dist.P2POp(dist.irecv, recv_low, prev, self.group, TAG_LOW))
            if recv_high is not None:
                ops.append(dist.P2POp(dist.irecv, recv_high, nxt, self.group, TAG_HIGH))
            import torch
            ctx = torch.cuda.stream(stream) if (stream is not None and flat.is_cuda) else _null()
            with ctx:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            if recv_low is not None:
                self.packer.unpack(flat, layout, fb["low_halo"], recv_low, stream)
            if recv_high is not None:
                self.packer.unpack(flat, layout, fb["high_halo"], recv_high, stream)


class GridArray:
    """This rank's block of an array decomposed over a ``CartGrid``."""

    def __init__(self, grid: CartGrid, dtype="float32", group=None, exchanger=None):
        from .runtime import HaloArray
        self.grid = grid
        self.block = HaloArray(grid.local_shape, grid.lo, grid.hi, dtype)
        self.exchanger = exchanger or GridExchanger(grid, group)
        self.rank = self.exchanger.rank

    def halo_transfer(self, stream=None) -> None:
        self.exchanger.exchange(self.block.data, self.block.layout, stream)


class GridStepper:
    """Fused step on a grid block: kernel (local dims' images refreshed in its
    epilogue), then the decomposed dims' faces, ascending."""

    def __init__(self, kernel, arr: GridArray, scalars=None):
        self.kernel = kernel
        self.arr = arr
        self.scalars = scalars
        self._remote = sum(1 << d for d, s in enumerate(arr.grid.splits) if s > 1)

    def step(self) -> None:
        from .runtime import step
        blk = self.arr.block
        step(self.kernel, blk, self.scalars, wrap_mask=self.arr.grid.local_mask)
        if self._remote:
            self.arr.exchanger.exchange(blk.data, blk.layout, dims=self._remote)

    def iterate(self, steps: int) -> None:
        from .runtime import launch
        if steps <= 0:
            return
        self.arr.halo_transfer()
        for _ in range(steps - 1):
            self.step()
        launch(self.kernel, [self.arr.block], None, self.scalars)


class MultiGrid:
    """All images of a ``CartGrid`` on one GPU, faces moved with ``lope_copy_box``
    between the blocks in the exchange order: the grid pipeline checked against a
    single-block run without needing more GPUs."""

    def __init__(self, kernel, grid: CartGrid, dtype, scalars=None):
        from .runtime import HaloArray
        self.grid = grid
        self.kernel = kernel
        self.scalars = scalars
        self.blocks = [HaloArray(grid.local_shape, grid.lo, grid.hi, dtype) for _ in range(grid.nranks)]

    def set_global(self, field: np.ndarray) -> None:
        for r, b in enumerate(self.blocks):
            o = self.grid.origin(r)
            sl = tuple(slice(o[d], o[d] + self.grid.local_shape[d]) for d in range(field.ndim))
            b.set_interior(np.ascontiguousarray(field[sl]))

    def get_global(self) -> np.ndarray:
        out = np.empty(self.grid.global_shape, dtype=self.blocks[0].get_interior().dtype)
        for r, b in enumerate(self.blocks):
            o = self.grid.origin(r)
            sl = tuple(slice(o[d], o[d] + self.grid.local_shape[d]) for d in range(out.ndim))
            out[sl] = b.get_interior()
        return out

    def exchange(self, dims=None) -> None:
        from .runtime import halo_transfer
        L = self.blocks[0].layout
        for d in range(int(L.rank)):
            if dims is not None and not (dims >> d) & 1:
                continue
            if int(L.lo[d]) == 0 and int(L.hi[d]) == 0:
                continue
            if self.grid.splits[d] == 1:
                for b in self.blocks:
                    halo_transfer(b, dims_mask=1 << d)
                continue
            fb = face_boxes(L, d)
            # every block's two faces along d in one lope_copy_boxes launch (the halo slabs
            # written are never read within the same dim)
            items = []
            for r, b in enumerate(self.blocks):
                prev = self.blocks[self.grid.neighbour(r, d, -1)]
                nxt = self.blocks[self.grid.neighbour(r, d, +1)]
                for dst_box, src_blk, src_box in ((fb["low_halo"], prev, fb["last"]),
                                                  (fb["high_halo"], nxt, fb["first"])):
                    if dst_box[1][d] == 0:
                        continue
                    items.append((b.data.data_ptr(), src_blk.data.data_ptr(), dst_box[0], src_box[0], dst_box[1]))
            if items:
                n = len(items)
                _lib.check(_lib.lib().lope_copy_boxes(
                    ctypes.byref(L), n, (ctypes.c_void_p * n)(*[it[0] for it in items]),
                    (ctypes.c_void_p * n)(*[it[1] for it in items]),
                    (ctypes.c_int64 * (3 * n))(*[int(v) for it in items for v in it[2]]),
                    (ctypes.c_int64 * (3 * n))(*[int(v) for it in items for v in it[3]]),
                    (ctypes.c_int64 * (3 * n))(*[int(v) for it in items for v in it[4]]),
                    _stream_ptr(None)), "lope_copy_boxes")

    def step(self) -> None:
        from .runtime import step
        for b in self.blocks:
            step(self.kernel, b, self.scalars, wrap_mask=self.grid.local_mask)
        remote = sum(1 << d for d, s in enumerate(self.grid.splits) if s > 1)
        if remote:
            self.exchange(dims=remote)

    def iterate(self, steps: int) -> None:
        from .runtime import launch
        if steps <= 0:
            return
        self.exchange()
        for _ in range(steps - 1):
            self.step()
        for b in self.blocks:
            launch(self.kernel, [b], None, self.scalars)


# ---------------------------------------------------------------------------
# Fused exchange: the stencil kernel stores boundary planes into the neighbours'
# halos through NVLink peer memory (lope_step_planes_peer + CUDA IPC)


def _step_planes_peer(kernel, layout, src, dst, b, e, rs, is_, mask, lo_peer, hi_peer, stream):
    _lib.check(_lib.lib().lope_step_planes_peer(kernel.handle, ctypes.byref(layout), ctypes.c_void_p(src),
                                                ctypes.c_void_p(dst), b, e, rs, is_, mask,
                                                ctypes.c_void_p(lo_peer), ctypes.c_void_p(hi_peer),
                                                _stream_ptr(stream)), "lope_step_planes_peer")


class PeerMultiSlab:
    """P slabs on one GPU with the fused exchange: each block's kernel stores its
    boundary planes' images straight into the neighbouring blocks' halos, so a step
    is P kernels and no exchange at all.  Checks the peer-store epilogue against the
    undecomposed run (the multi-GPU version maps the neighbours through CUDA IPC)."""

    def __init__(self, kernel, global_shape, lo, hi, dtype, nranks: int, scalars=None):
        from .runtime import HaloArray
        self.grid = SlabGrid(global_shape, nranks, lo, hi)
        self.kernel = kernel
        self.scalars = scalars
        self.blocks = [HaloArray(self.grid.local_shape, lo, hi, dtype) for _ in range(nranks)]
        for b in self.blocks:
            b.spare()
        self.dim = len(global_shape) - 1
        self._rs, self._is = kernel.scalar_args(scalars)

    set_global = MultiSlab.set_global
    get_global = MultiSlab.get_global
    _mask = MultiSlab._mask
    halo_transfer = MultiSlab.halo_transfer

    def step(self) -> None:
        P = len(self.blocks)
        L = self.blocks[0].layout
        m = int(L.interior[self.dim])
        full = (1 << len(self.grid.global_shape)) - 1
        outs = [b.spare().data_ptr() for b in self.blocks]
        for r, b in enumerate(self.blocks):
            lo_peer = outs[(r - 1) % P] if P > 1 else 0
            hi_peer = outs[(r + 1) % P] if P > 1 else 0
            _step_planes_peer(self.kernel, b.layout, b.data.data_ptr(), outs[r], 0, m, self._rs, self._is,
                              full, lo_peer, hi_peer, None)
        for b in self.blocks:
            b.swap()

    def iterate(self, steps: int) -> None:
        from .runtime import launch
        if steps <= 0:
            return
        self.halo_transfer()
        for _ in range(steps - 1):
            self.step()
        for b in self.blocks:
            launch(self.kernel, [b], None, self.scalars)


class SlabComm:
    """This image's communicator in liblope_b200.so (``lope_comm``, include/lope_b200.h).

    The exchange of ``Machine._halo_exchange`` (runtime.py:643-711) between slab images
    lives behind the C ABI: ``exchange`` (HALO_TRANSFER), ``step`` (one fused stencil
    kernel whose epilogue stores the boundary planes' images into the neighbours' blocks,
    ordered against the neighbours by stream memory operations on peer flags) and
    ``sync``.  Python only moves the setup records between ranks (``gather``: any
    all-gather of bytes in rank order; ``torch.distributed.all_gather_object`` for one
    process per GPU) -- nothing in the step loop.
    """

    def __init__(self, block, rank: int, nranks: int):
        block.spare()                        # both ping-pong buffers exist, fixed indices
        self.block = block
        self.rank, self.nranks = int(rank), int(nranks)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().lope_comm_create(self.nranks, self.rank, ctypes.byref(h)), "lope_comm_create")
        self.handle = h.value

    def export(self) -> bytes:
        n = _lib.lib().lope_comm_record_size()
        rec = ctypes.create_string_buffer(n)
        b = self.block
        _lib.check(_lib.lib().lope_comm_export(self.handle, ctypes.byref(b.layout),
                                               ctypes.c_void_p(b._bufs[0].data_ptr()),
                                               ctypes.c_void_p(b._bufs[1].data_ptr()), rec), "lope_comm_export")
        return bytes(rec.raw)

    def connect(self, records: Sequence[bytes]) -> None:
        blob = b"".join(records)
        _lib.check(_lib.lib().lope_comm_connect(self.handle, blob), "lope_comm_connect")

    def nccl_init(self, uid: bytes) -> None:
        _lib.check(_lib.lib().lope_comm_nccl_init(self.handle, uid), "lope_comm_nccl_init")

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.lib().lope_comm_nccl_unique_id(buf), "lope_comm_nccl_unique_id")
        return bytes(buf.raw)

    def info(self):
        r, n, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        e = ctypes.c_uint32()
        _lib.check(_lib.lib().lope_comm_info(self.handle, ctypes.byref(r), ctypes.byref(n), ctypes.byref(e),
                                             ctypes.byref(t)), "lope_comm_info")
        return {"rank": r.value, "nranks": n.value, "epoch": e.value,
                "transport": {0: None, 1: "peer", 2: "nccl", 3: "peer-host-ordered"}[t.value]}

    def exchange(self, dims_mask: Optional[int] = None, stream=None, live: Optional[int] = None) -> None:
        mask = (1 << self.block.rank) - 1 if dims_mask is None else dims_mask
        _lib.check(_lib.lib().lope_halo_exchange(self.handle, self.block._live if live is None else live, mask,
                                                 _stream_ptr(stream)), "lope_halo_exchange")

    def exchange_begin(self, dims_mask: Optional[int] = None, stream=None) -> None:
        mask = (1 << self.block.rank) - 1 if dims_mask is None else dims_mask
        _lib.check(_lib.lib().lope_halo_exchange_begin(self.handle, self.block._live, mask, _stream_ptr(stream)),
                   "lope_halo_exchange_begin")

    def exchange_end(self, stream=None) -> None:
        _lib.check(_lib.lib().lope_halo_exchange_end(self.handle, _stream_ptr(stream)), "lope_halo_exchange_end")

    def step(self, kernel, rs, is_, stream=None) -> None:
        _lib.check(_lib.lib().lope_comm_step(self.handle, kernel.handle, self.block._live, rs, is_,
                                             _stream_ptr(stream)), "lope_comm_step")
        self.block.swap()

    def sync(self, stream=None) -> None:
        _lib.check(_lib.lib().lope_comm_sync(self.handle, _stream_ptr(stream)), "lope_comm_sync")

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib().lope_comm_destroy(ctypes.c_void_p(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerSlabStepper:
    """Multi-GPU slabs with the exchange fused into the kernel (one process per GPU),
    through the C-ABI communicator (``SlabComm`` / ``lope_comm``).

    A step is ``lope_comm_step``: a stream wait on the two neighbours' step flags, ONE
    kernel that writes the slab's interior, the periodic images of the non-decomposed
    dims and its boundary planes' images straight into the neighbours' output blocks
    over NVLink, and the flag writes -- no collective and no host synchronisation.
    ``torch.distributed`` only carries the setup records (all ranks agree: a rank that
    cannot export or map makes every rank raise, and the caller falls back together).
    """

    def __init__(self, kernel, arr: SlabArray, scalars=None, group=None):
        import torch.distributed as dist
        self.kernel = kernel
        self.arr = arr
        self.scalars = scalars
        self.group = group
        self.dist = dist
        self._rs, self._is = kernel.scalar_args(scalars)
        blk = arr.block
        self.rank, self.size = arr.rank, arr.size
        self.comm, why = None, None
        rec = None
        try:
            self.comm = SlabComm(blk, self.rank, self.size)
            rec = self.comm.export()
        except Exception as e:          # pragma: no cover - depends on the allocator
            why = repr(e)
        allr = [None] * self.size
        dist.all_gather_object(allr, rec, group=group)
        ok = 0
        if all(r is not None for r in allr):
            try:
                self.comm.connect(allr)
                ok = 1
            except Exception as e:      # pragma: no cover - depends on the node
                why = repr(e)
        flags = [None] * self.size
        dist.all_gather_object(flags, ok, group=group)
        if not all(flags):
            self.close()
            raise RuntimeError(f"peer mapping failed on some rank ({why or 'another rank'})")
        self.full = (1 << blk.rank) - 1
        self.m = int(blk.layout.interior[arr.dim])
        # two processes on one GPU (tests): no device-side waits between them, the host
        # orders every operation instead (synchronise + barrier)
        self.host_ordered = self.comm.info()["transport"] == "peer-host-ordered"

    def close(self) -> None:
        if self.comm is not None:
            self.comm.close()
            self.comm = None

    def _host_order(self) -> None:
        if self.host_ordered:
            import torch
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)

    def barrier(self) -> None:
        """Order this rank's stream after both neighbours' latest operation."""
        self.comm.sync()
        self._host_order()

    def exchange(self) -> None:
        """``HALO_TRANSFER``: local dims wrap on the GPU, the decomposed dim's halo
        planes are copied from the neighbours' live blocks (peer memory)."""
        self.comm.exchange_begin()
        self._host_order()
        self.comm.exchange_end()
        self._host_order()

    def tune(self) -> int:
        """Run real steps until the plan for this block is chosen; returns the count."""
        n = 0
        while self.kernel.tuning(self.arr.block, self.full):
            self.step()
            n += 1
        return n

    def step(self) -> None:
        blk = self.arr.block
        tuner = self.kernel.tuner(blk, self.full)
        if tuner is not None:
            tuner.before()
        self.comm.step(self.kernel, self._rs, self._is)
        self._host_order()
        if tuner is not None:
            tuner.after()

    def iterate(self, steps: int) -> None:
        from .runtime import launch
        if steps <= 0:
            return
        self.exchange()
        for _ in range(steps - 1):
            self.step()
        self.barrier()
        launch(self.kernel, [self.arr.block], None, self.scalars)


class CommMultiSlab:
    """P slab images in ONE process, each with its own ``lope_comm`` and CUDA stream,
    connected through raw pointers: the C-ABI exchange and fused-step protocol (flags,
    stream waits, peer stores) exercised end to end on one GPU.

    Nothing here waits inside a kernel: the waits are stream memory operations, and the
    operations are enqueued round by round (every image's operation k before any image's
    operation k+1), so each wait's signal is enqueued before it -- no order of the
    streams on the hardware queues can deadlock.  Run it with
    ``CUDA_DEVICE_MAX_CONNECTIONS`` >= P + 1 so the streams do not share a queue.
    """

    def __init__(self, kernel, global_shape, lo, hi, dtype, nranks: int, scalars=None):
        import torch
        from .runtime import HaloArray
        self.grid = SlabGrid(global_shape, nranks, lo, hi)
        self.kernel = kernel
        self.scalars = scalars
        self.blocks = [HaloArray(self.grid.local_shape, lo, hi, dtype) for _ in range(nranks)]
        self.streams = [torch.cuda.Stream() for _ in range(nranks)]
        torch.cuda.synchronize()
        self.comms = [SlabComm(b, r, nranks) for r, b in enumerate(self.blocks)]
        torch.cuda.synchronize()
        recs = [c.export() for c in self.comms]
        for c in self.comms:
            c.connect(recs)
        self._rs, self._is = kernel.scalar_args(scalars)
        self.dim = len(global_shape) - 1

    set_global = MultiSlab.set_global
    get_global = MultiSlab.get_global

    def _all(self, fn):
        import torch
        for c, s in zip(self.comms, self.streams):
            with torch.cuda.stream(s):
                fn(c, s)

    def halo_transfer(self) -> None:
        # two rounds: every image's "ready" signal is enqueued before any image waits
        self._all(lambda c, s: c.exchange_begin(stream=s))
        self._all(lambda c, s: c.exchange_end(stream=s))

    def step(self) -> None:
        self._all(lambda c, s: c.step(self.kernel, self._rs, self._is, stream=s))

    def iterate(self, steps: int) -> None:
        import torch
        from .runtime import launch
        if steps <= 0:
            return
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        self.halo_transfer()
        for _ in range(steps - 1):
            self.step()
        self._all(lambda c, s: c.sync(stream=s))
        self._all(lambda c, s: launch(self.kernel, [c.block], None, self.scalars, stream=s))
        for s in self.streams:
            cur.wait_stream(s)

    def close(self) -> None:
        for c in self.comms:
            c.close()
