"""Slab decomposition and the ring face exchange, on CPU with the gloo backend.

Each rank holds its slab in the exact device layout (``lope_layout_init``) as a
CPU tensor and runs the same ``NcclExchanger`` code the GPUs run over NCCL; the
result must equal the reference exchange (``runtime.py:643-711``) cell for cell,
as restated by ``oracle.exchange_blocks`` (itself pinned to the reference's
blocks in tests/golden/exchange.npz).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lope_oracle as O
from paper_1502_03504_b200 import _lib
from paper_1502_03504_b200.diagnostics import RuntimeFault
from paper_1502_03504_b200.dist import NcclExchanger, SlabGrid, faces


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def padded_to_flat(padded, layout):
    """Place a numpy padded block (reference index order) into a flat device-layout array."""
    L = layout
    flat = np.zeros(L.count, dtype=padded.dtype)
    idx = np.indices(padded.shape).reshape(padded.ndim, -1)
    strides = [1, L.stride[1], L.stride[2]][: padded.ndim]
    lin = L.base + sum(i * s for i, s in zip(idx, strides))
    flat[lin] = padded.reshape(-1)
    return flat


def flat_to_padded(flat, layout, shape):
    L = layout
    idx = np.indices(shape).reshape(len(shape), -1)
    strides = [1, L.stride[1], L.stride[2]][: len(shape)]
    lin = L.base + sum(i * s for i, s in zip(idx, strides))
    return np.asarray(flat)[lin].reshape(shape)


def _worker(rank, size, port, gshape, lo, hi, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        grid = SlabGrid(gshape, size, lo, hi)
        field = O.hash_field(gshape, 99, np.float64)
        n = grid.local_shape[-1]
        part = field[..., rank * n:(rank + 1) * n]
        blk = O.embed(part, lo, hi)
        # local (non-decomposed) dims wrap on the device first; restated here on the host
        O.halo_fill(blk, lo, hi, dims=tuple(range(len(gshape) - 1)))
        L = _lib.make_layout(len(gshape), "f64", grid.local_shape, lo, hi)
        flat = torch.from_numpy(padded_to_flat(blk, L))
        NcclExchanger().exchange(flat, L)
        got = flat_to_padded(flat.numpy(), L, blk.shape)
        # reference: every image's padded block after one exchange
        blocks = [O.embed(field[..., k * n:(k + 1) * n], lo, hi) for k in range(size)]
        O.exchange_blocks(blocks, lo, hi, axis=-1)
        q.put((rank, bool(np.array_equal(got, blocks[rank]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size,gshape,lo,hi", [
    (2, (8, 12), (1, 1), (1, 1)),
    (2, (6, 8), (2, 2), (1, 2)),
    (3, (5, 9), (1, 0), (2, 1)),
    (2, (4, 5, 8), (1, 1, 1), (1, 1, 1)),
    (4, (4, 3, 8), (0, 1, 2), (1, 0, 2)),
])
def test_gloo_ring_exchange_matches_reference(size, gshape, lo, hi):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, gshape, lo, hi, q)) for r in range(size)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(size))
    for p in procs:
        p.join(timeout=60)
    assert all(results.values()), results


def test_single_rank_exchange_wraps_locally():
    gshape, lo, hi = (6, 5, 4), (1, 1, 2), (1, 2, 1)
    field = O.hash_field(gshape, 5, np.float64)
    blk = O.embed(field, lo, hi)
    O.halo_fill(blk, lo, hi, dims=(0, 1))
    L = _lib.make_layout(3, "f64", gshape, lo, hi)
    flat = torch.from_numpy(padded_to_flat(blk, L))
    f = faces(flat, L)
    f["low_halo"].copy_(f["last"])
    f["high_halo"].copy_(f["first"])
    want = O.embed(field, lo, hi)
    O.halo_fill(want, lo, hi)
    assert np.array_equal(flat_to_padded(flat.numpy(), L, blk.shape), want)


def test_slab_grid_checks_and_neighbours():
    g = SlabGrid((8, 16), 4, (1, 1), (1, 1))
    assert g.local_shape == (8, 4)
    assert g.origin(2) == (0, 8)
    assert g.neighbours(0) == (3, 1) and g.neighbours(3) == (2, 0)
    with pytest.raises(RuntimeFault) as e:
        SlabGrid((8, 10), 4, (1, 1), (1, 1))
    assert e.value.code == "E201"
    with pytest.raises(RuntimeFault) as e:
        SlabGrid((8, 4), 4, (2, 2), (2, 2))            # per-image extent 1 < halo 2 (F8)
    assert e.value.code == "E108"


def test_face_spans_address_whole_planes():
    L = _lib.make_layout(2, "f32", (10, 6), (1, 2), (1, 1))
    flat = torch.arange(L.count, dtype=torch.float32)
    f = faces(flat, L)
    assert f["low_halo"].numel() == 2 * L.stride[1]
    assert f["high_halo"].numel() == 1 * L.stride[1]
    assert f["first"].numel() == 1 * L.stride[1] and f["last"].numel() == 2 * L.stride[1]
    assert int(f["first"][0]) == 2 * L.stride[1]
    assert int(f["last"][0]) == 6 * L.stride[1]


# ---------------------------------------------------------------------------
# General process grids (MP x NP, P0 x P1 x P2): GridExchanger over gloo


class TorchCpuPacker:
    """Test-side face staging for CPU tensors (the GPUs use lope_box_pack/unpack)."""

    @staticmethod
    def _view(flat, L):
        r = int(L.rank)
        p = [int(L.padded[i]) if i < r else 1 for i in range(3)]
        s1 = int(L.stride[1]) if r > 1 else p[0]
        s2 = int(L.stride[2]) if r > 2 else s1 * p[1]
        return torch.as_strided(flat, size=tuple(p), stride=(1, s1, s2), storage_offset=int(L.base))

    def _box(self, flat, L, box):
        (b, e) = box
        v = self._view(flat, L)
        return v[b[0]:b[0] + e[0], b[1]:b[1] + e[1], b[2]:b[2] + e[2]]

    @staticmethod
    def alloc(flat, box):
        return torch.empty(int(np.prod(box[1])), dtype=flat.dtype)

    def pack(self, flat, L, box, stream=None):
        return self._box(flat, L, box).permute(2, 1, 0).reshape(-1).clone()

    def unpack(self, flat, L, box, buf, stream=None):
        e = box[1]
        self._box(flat, L, box).copy_(buf.reshape(e[2], e[1], e[0]).permute(2, 1, 0))

    def local_wrap(self, flat, L, d, stream=None):
        from paper_1502_03504_b200.dist import face_boxes
        fb = face_boxes(L, d)
        if int(L.lo[d]):
            self.unpack(flat, L, fb["low_halo"], self.pack(flat, L, fb["last"]))
        if int(L.hi[d]):
            self.unpack(flat, L, fb["high_halo"], self.pack(flat, L, fb["first"]))


def periodic_padded(field, origin, local, lo, hi):
    """The periodic global field over a block's padded window."""
    idx = [np.arange(o - l, o + m + h) % n for o, m, l, h, n in zip(origin, local, lo, hi, field.shape)]
    return field[np.ix_(*idx)]


def _grid_worker(rank, size, port, gshape, splits, lo, hi, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from paper_1502_03504_b200.dist import CartGrid, GridExchanger
        grid = CartGrid(gshape, splits, lo, hi)
        field = O.hash_field(gshape, 17, np.float64)
        o = grid.origin(rank)
        part = field[tuple(slice(o[d], o[d] + grid.local_shape[d]) for d in range(len(gshape)))]
        blk = O.embed(part, lo, hi)
        L = _lib.make_layout(len(gshape), "f64", grid.local_shape, lo, hi)
        flat = torch.from_numpy(padded_to_flat(blk, L))
        GridExchanger(grid, packer=TorchCpuPacker()).exchange(flat, L)
        got = flat_to_padded(flat.numpy(), L, blk.shape)
        want = periodic_padded(field, o, grid.local_shape, lo, hi)
        q.put((rank, bool(np.array_equal(got, want))))
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("gshape,splits,lo,hi", [
    ((8, 12), (2, 2), (1, 1), (1, 1)),        # reference images=4, grid_rows=2
    ((9, 8), (3, 2), (2, 1), (1, 2)),         # images=6, grid_rows=2, asymmetric halos
    ((8, 6), (4, 1), (1, 1), (1, 1)),         # images=4, grid_rows=1: dim 1 only (strided faces)
    ((6, 4, 8), (1, 2, 2), (1, 1, 1), (1, 1, 1)),
    ((4, 6, 4), (2, 2, 1), (1, 0, 2), (2, 1, 0)),
])
def test_gloo_grid_exchange_fills_periodic_images(gshape, splits, lo, hi):
    size = int(np.prod(splits))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, size, port, gshape, splits, lo, hi, q))
             for r in range(size)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(size))
    for p in procs:
        p.join(timeout=60)
    assert all(v is True for v in results.values()), results


def test_cart_grid_matches_reference_image_order():
    """Image k (1-based) of RunConfig(images=P, grid_rows=MP) sits at (pcol, prow) =
    ((k-1) div MP, (k-1) mod MP) (grid.py:27-33) and neighbours wrap cyclically."""
    from paper_1502_03504_b200.dist import CartGrid
    g = CartGrid.from_images((12, 8), 6, 2, (1, 1), (1, 1))
    assert g.splits == (3, 2) and g.local_shape == (4, 4)
    for k in range(1, 7):
        prow, pcol = (k - 1) % 2, (k - 1) // 2
        assert g.coords(k - 1) == (pcol, prow)
        assert g.origin(k - 1) == (pcol * 4, prow * 4)
    assert g.neighbour(0, 0, -1) == 4 and g.neighbour(0, 1, -1) == 1
    assert g.local_mask == 0
    assert CartGrid((8, 6), (1, 3), (1, 1), (1, 1)).local_mask == 1
    with pytest.raises(RuntimeFault) as e:
        CartGrid.from_images((12, 8), 6, 4, (1, 1), (1, 1))
    assert e.value.code == "E201"
    with pytest.raises(RuntimeFault) as e:
        CartGrid((12, 9), (2, 2), (1, 1), (1, 1))
    assert e.value.code == "E201"
