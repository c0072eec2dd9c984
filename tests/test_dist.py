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
