"""Slab-decomposed pipeline on one GPU: P in-process slabs (boundary planes, face
spans, ring exchange) must give bit-identical fields to the undecomposed run, the
reference's decomposition invariance (tests/test_runtime.py:90-98 there)."""

import numpy as np
import pytest

from oracle import lope_oracle as O
from paper_1502_03504_b200 import stencils

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1502_03504_b200 import dist as D  # noqa: E402
from paper_1502_03504_b200 import runtime as R  # noqa: E402


def halos(kir):
    fp = kir.footprints[kir.array_params[0]].dims
    return [n for n, _ in fp], [p for _, p in fp]


@pytest.mark.parametrize("name,shape,dt,ps", [
    ("lap3d7", (64, 40, 48), "float32", (2, 3, 4, 8)),
    ("box5x5", (96, 64), "float64", (2, 4, 8)),
    ("drift2", (64, 48), "float32", (2, 4)),
    ("heat2d", (256, 128), "float64", (2, 4, 8)),
])
def test_slab_decomposition_is_bitwise_invariant(name, shape, dt, ps):
    kir = stencils.by_name(name)
    lo, hi = halos(kir)
    npdt = np.float32 if dt == "float32" else np.float64
    sc = {"c": 0.25} if name == "drift2" else None
    field = O.hash_field(shape, 31, npdt)
    k = R.CompiledKernel(kir, dt)
    base = R.HaloArray(shape, lo, hi, dt)
    base.set_interior(field)
    R.iterate(k, base, 5, sc)
    want = base.get_interior()
    ref = field
    for _ in range(5):
        ref = O.periodic_apply(ref, kir, sc, npdt)
    assert O.equal_bits(want, ref)
    for p in ps:
        ms = D.MultiSlab(k, shape, lo, hi, dt, p, sc)
        ms.set_global(field)
        ms.iterate(5)
        got = ms.get_global()
        assert O.equal_bits(got, want), (name, p, O.first_mismatch(got, want))


def test_single_rank_stepper_matches_runtime():
    kir = stencils.lap3d7()
    shape = (128, 64, 32)
    field = O.hash_field(shape, 3, np.float32)
    k = R.CompiledKernel(kir, "float32")
    arr = D.SlabArray(shape, (1, 1, 1), (1, 1, 1), "float32")
    arr.block.set_interior(field)
    D.SlabStepper(k, arr).iterate(4)
    ref = field
    for _ in range(4):
        ref = O.periodic_apply(ref, kir, None, np.float32)
    assert O.equal_bits(arr.block.get_interior(), ref)


@pytest.mark.parametrize("name,shape,dt,grids", [
    ("box5x5", (96, 64), "float64", [(2, 2), (4, 1), (1, 4), (3, 2)]),
    ("ninept2d", (256, 96), "float32", [(2, 2), (8, 1), (2, 3)]),
    ("drift2", (64, 48), "float32", [(2, 2), (4, 2)]),
    ("lap3d7", (64, 40, 48), "float32", [(2, 2, 2), (1, 2, 4), (2, 1, 1), (4, 2, 1)]),
])
def test_grid_decomposition_is_bitwise_invariant(name, shape, dt, grids):
    """MP x NP (and 3-D) image grids: every block computes and exchanges faces in the
    reference's dim order; the gathered field equals the undecomposed run's bits."""
    kir = stencils.by_name(name)
    lo, hi = halos(kir)
    npdt = np.float32 if dt == "float32" else np.float64
    sc = {"c": 0.25} if name == "drift2" else None
    field = O.hash_field(shape, 41, npdt)
    k = R.CompiledKernel(kir, dt)
    base = R.HaloArray(shape, lo, hi, dt)
    base.set_interior(field)
    R.iterate(k, base, 4, sc)
    want = base.get_interior()
    for splits in grids:
        mg = D.MultiGrid(k, D.CartGrid(shape, splits, lo, hi), dt, sc)
        mg.set_global(field)
        mg.iterate(4)
        got = mg.get_global()
        assert O.equal_bits(got, want), (name, splits, O.first_mismatch(got, want))


def test_grid_exchange_blocks_hold_periodic_images():
    """After one exchange every padded cell of every block is its periodic image."""
    shape, lo, hi = (48, 36, 20), (1, 2, 1), (2, 1, 1)
    field = O.hash_field(shape, 43, np.float64)
    k = R.CompiledKernel(stencils.lap3d7(), "float64")
    g = D.CartGrid(shape, (2, 3, 2), lo, hi)
    mg = D.MultiGrid(k, g, "float64")
    mg.set_global(field)
    mg.exchange()
    for r, b in enumerate(mg.blocks):
        o = g.origin(r)
        idx = [np.arange(o[d] - lo[d], o[d] + g.local_shape[d] + hi[d]) % shape[d] for d in range(3)]
        assert np.array_equal(b.get_padded(), field[np.ix_(*idx)]), r


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_box_pack_unpack_round_trip(dt):
    """lope_box_pack gathers a box column-major; lope_box_unpack scatters it back."""
    shape, lo, hi = (37, 21, 9), (2, 1, 3), (1, 2, 2)
    npdt = np.float32 if dt == "float32" else np.float64
    arr = R.HaloArray(shape, lo, hi, dt)
    arr.fill_hash(5)
    R.halo_transfer(arr)
    padded = arr.get_padded()
    L = arr.layout
    rng = np.random.default_rng(1)
    for _ in range(12):
        e = [int(rng.integers(1, p + 1)) for p in padded.shape]
        b = [int(rng.integers(0, p - w + 1)) for p, w in zip(padded.shape, e)]
        box = (tuple(b), tuple(e))
        buf = D.DevicePacker().pack(arr.data, L, box)
        want = padded[b[0]:b[0] + e[0], b[1]:b[1] + e[1], b[2]:b[2] + e[2]].reshape(-1, order="F")
        assert np.array_equal(buf.cpu().numpy(), want.astype(npdt))
        dst = R.HaloArray(shape, lo, hi, dt)
        D.DevicePacker().unpack(dst.data, L, box, buf)
        got = dst.get_padded()
        ref = np.zeros_like(padded)
        ref[b[0]:b[0] + e[0], b[1]:b[1] + e[1], b[2]:b[2] + e[2]] = padded[b[0]:b[0] + e[0], b[1]:b[1] + e[1],
                                                                           b[2]:b[2] + e[2]]
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("name,shape,dt,ps", [
    ("lap3d7", (64, 40, 48), "float32", (1, 2, 3, 4)),
    ("box5x5", (96, 64), "float64", (2, 4)),
    ("heat2d", (256, 96), "float64", (3,)),
    ("drift2", (64, 48), "float32", (2,)),
])
def test_fused_peer_exchange_is_bitwise_invariant(name, shape, dt, ps):
    """Kernels that store their boundary planes into the neighbouring blocks' halos
    (lope_step_planes_peer) need no exchange step and give the undecomposed bits."""
    kir = stencils.by_name(name)
    lo, hi = halos(kir)
    npdt = np.float32 if dt == "float32" else np.float64
    sc = {"c": 0.25} if name == "drift2" else None
    field = O.hash_field(shape, 37, npdt)
    k = R.CompiledKernel(kir, dt)
    base = R.HaloArray(shape, lo, hi, dt)
    base.set_interior(field)
    R.iterate(k, base, 5, sc)
    want = base.get_interior()
    for p in ps:
        ms = D.PeerMultiSlab(k, shape, lo, hi, dt, p, sc)
        ms.set_global(field)
        ms.iterate(5)
        got = ms.get_global()
        assert O.equal_bits(got, want), (name, p, O.first_mismatch(got, want))


def _peer_worker(rank, size, port, q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        kir = stencils.lap3d7()
        gshape = (64, 32, 16 * size)
        field = O.hash_field(gshape, 51, np.float32)
        k = R.CompiledKernel(kir, "float32")
        arr = D.SlabArray((64, 32, 16), (1, 1, 1), (1, 1, 1), "float32")
        arr.block.set_interior(np.ascontiguousarray(field[..., rank * 16:(rank + 1) * 16]))
        st = D.PeerSlabStepper(k, arr)
        st.iterate(6)
        torch.cuda.synchronize()
        got = arr.block.get_interior()
        want = field
        for _ in range(6):
            want = O.periodic_apply(want, kir, None, np.float32)
        ok = O.equal_bits(got, want[..., rank * 16:(rank + 1) * 16])
        dist.barrier()
        st.close()
        q.put((rank, bool(ok)))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_fused_peer_exchange_across_processes_via_ipc():
    """Two processes (one GPU here, one per GPU in production) map each other's
    blocks with CUDA IPC; the fused kernels write across the process boundary."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(v is True for v in res.values()), res
