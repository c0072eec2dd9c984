"""GPU parity of the shapes that used to fall off the TMA path.

* ragged x: interiors that are not a whole number of 16-byte vectors (and narrower than
  two 64-byte atoms), sub-range launches whose start and end are not vector aligned --
  the tiled kernel masks the straddling vectors and stores x images cell by cell;
* rank 1 (``corpus/avg3.lope``): the vector row kernel;
* kernels over several arrays: the fused step (``lope_step_arrays``) stores every
  stored array's periodic images from the multi-array TMA kernel.

Every case runs through the C ABI, is compared bit for bit with the oracle (fp64 = the
reference's own arithmetic, pinned by tests/test_oracle.py; fp32 = its restatement) and
asserts from the kernel's launch counters which kernel family actually ran.
"""

import json

import numpy as np
import pytest

from oracle import lope_oracle as O
from paper_1502_03504_b200 import stencils
from paper_1502_03504_b200.ir import KernelBuilder, deserialize

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1502_03504_b200 import runtime as R  # noqa: E402

NP = {"float32": np.float32, "float64": np.float64}


def launches(k):
    return json.loads(k.describe())["launches"]


def halos(kir, a=0):
    fp = kir.footprints[kir.array_params[a]].dims
    return [n for n, _ in fp], [p for _, p in fp]


@pytest.mark.parametrize("name,shape,dt", [
    ("lap3d7", (1001, 37, 19), "float32"),
    ("lap3d7", (13, 30, 9), "float32"),       # narrower than two atoms: exact x images
    ("lap3d7", (77, 21, 11), "float64"),
    ("heat2d", (1023, 65), "float32"),
    ("heat2d", (6, 40), "float32"),
    ("ninept2d", (333, 47), "float64"),
    ("box5x5", (101, 33), "float64"),
    ("box5x5", (9, 12), "float32"),
])
def test_ragged_x_runs_tiled_and_matches_the_oracle(monkeypatch, name, shape, dt):
    monkeypatch.setenv("LOPE_AUTOTUNE", "0")
    monkeypatch.setenv("LOPE_NO_TBLOCK", "1")       # the fused single steps themselves
    kir = stencils.by_name(name)
    k = R.CompiledKernel(kir, dt)
    lo, hi = halos(kir)
    field = O.hash_field(shape, 11, NP[dt])
    arr = R.HaloArray(shape, lo, hi, dt)
    arr.set_interior(field)
    R.iterate(k, arr, 4)
    got = arr.get_padded()
    want = O.machine_run(field, kir, 4, None, NP[dt], lo, hi)
    assert O.equal_bits(got, want), O.first_mismatch(got, want)
    n = launches(k)
    assert n["tiled"] >= 4 and n["generic"] == 0, n


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_unaligned_subrange_launches_run_tiled(dt):
    """Launch ranges starting and ending inside a vector: the cells of the straddling
    vectors outside the range keep the snapshot's values (copy-through)."""
    rng = np.random.default_rng(5)
    for name, shape in (("lap3d7", (70, 23, 9)), ("heat2d", (205, 31)), ("box5x5", (66, 20))):
        kir = stencils.by_name(name)
        k = R.CompiledKernel(kir, dt)
        lo, hi = halos(kir)
        field = O.hash_field(shape, 3, NP[dt])
        for _ in range(6):
            ranges = []
            for m in shape:
                a = int(rng.integers(1, m // 2))
                b = int(rng.integers(a, m + 1))
                ranges.append((a, b))
            arr = R.HaloArray(shape, lo, hi, dt)
            arr.set_interior(field)
            R.halo_transfer(arr)
            R.launch(k, [arr], ranges)
            blk = O.embed(field, lo, hi, NP[dt])
            O.halo_fill(blk, lo, hi)
            O.launch({kir.array_params[0]: blk}, {kir.array_params[0]: (lo, hi)}, kir, ranges, None, NP[dt])
            got = arr.get_padded()
            assert O.equal_bits(got, blk), (name, ranges, O.first_mismatch(got, blk))
        assert launches(k)["generic"] == 0


def test_random_kernels_on_ragged_x_tiled_equals_generic_and_oracle(monkeypatch, golden_random):
    """Every golden random kernel of rank 2/3 on x extents that are not whole vectors,
    asymmetric halos: tiled == generic (padded block) and == the oracle (interior)."""
    meta, _ = golden_random
    rng = np.random.default_rng(77)
    monkeypatch.setenv("LOPE_AUTOTUNE", "0")
    monkeypatch.setenv("LOPE_NO_TBLOCK", "1")
    checked = 0
    for m in meta:
        kir = deserialize(m["ir"])
        if kir.rank < 2:
            continue
        fp = kir.footprints[kir.array_params[0]].dims
        lo = [int(n) + int(rng.integers(0, 2)) for n, _ in fp]
        hi = [int(p) + int(rng.integers(0, 2)) for _, p in fp]
        for dt in ("float32", "float64"):
            mx = int(rng.integers(5, 200)) | 1           # odd: never a whole vector
            shape = (mx, int(rng.integers(9, 40))) + ((int(rng.integers(5, 15)),) if kir.rank == 3 else ())
            if any(s < l_ + h_ for s, l_, h_ in zip(shape, lo, hi)):
                continue
            field = O.hash_field(shape, int(m["trial"]) + 13, NP[dt])
            k = R.CompiledKernel(kir, dt)
            outs = []
            for generic in (False, True):
                if generic:
                    monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
                a = R.HaloArray(shape, lo, hi, dt)
                a.set_interior(field)
                R.iterate(k, a, 3, m["scalars"])
                outs.append(a.get_padded())
                monkeypatch.delenv("LOPE_FORCE_GENERIC", raising=False)
            assert O.equal_bits(outs[0], outs[1]), (m["trial"], dt, shape, lo, hi, m["source"])
            want = O.machine_run(field, kir, 3, m["scalars"], NP[dt], lo, hi)
            assert O.equal_bits(O.interior(outs[0], lo, hi), O.interior(want, lo, hi)), (m["trial"], dt, shape)
            n = launches(k)
            assert n["tiled"] > 0, n
            checked += 1
    assert checked >= 80


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_rank1_kernels_run_the_row_kernel(dt, golden_random):
    """corpus avg3 and every rank-1 golden random kernel: fused steps (images cell by
    cell), plain launches and unaligned sub-ranges on the row kernel == the oracle."""
    meta, _ = golden_random
    kirs = [(stencils.avg3(), None)] + [(deserialize(m["ir"]), m["scalars"]) for m in meta
                                        if deserialize(m["ir"]).rank == 1]
    assert len(kirs) >= 9
    rng = np.random.default_rng(8)
    for kir, sc in kirs:
        k = R.CompiledKernel(kir, dt)
        assert json.loads(k.describe())["path"] == "row"
        lo, hi = halos(kir)
        for n in (1, 7, 64, 1000, 4099):
            if n < lo[0] + hi[0]:
                continue
            field = O.hash_field((n,), n, NP[dt])
            arr = R.HaloArray((n,), lo, hi, dt)
            arr.set_interior(field)
            R.iterate(k, arr, 5, sc)
            want = O.machine_run(field, kir, 5, sc, NP[dt], lo, hi)
            got = arr.get_padded()
            assert O.equal_bits(got, want), (kir.name, n, O.first_mismatch(got, want))
            a = int(rng.integers(1, n + 1))
            b = int(rng.integers(a, n + 1))
            arr2 = R.HaloArray((n,), lo, hi, dt)
            arr2.set_interior(field)
            R.halo_transfer(arr2)
            R.launch(k, [arr2], [(a, b)], sc)
            blk = O.embed(field, lo, hi, NP[dt])
            O.halo_fill(blk, lo, hi)
            O.launch({kir.array_params[0]: blk}, {kir.array_params[0]: (lo, hi)}, kir, [(a, b)], sc, NP[dt])
            assert O.equal_bits(arr2.get_padded(), blk), (kir.name, n, a, b)
        nl = launches(k)
        assert nl["row"] > 0 and nl["generic"] == 0, nl


def _multi_kernel(rank, na):
    kb = KernelBuilder(f"fused{rank}{na}", rank)
    arrs = [kb.array(n) for n in "uvwx"[:na]]
    z = (0,) * rank

    def off(d, s_):
        o = [0] * rank
        o[d] = s_
        return tuple(o)

    e = arrs[0][z]
    for i, a in enumerate(arrs[1:], 1):
        e = e + (a[off(0, 1)] - a[off(rank - 1, -1)]) * (0.25 * i) + a[off(1, -1)] / 3.0
    kb.store(arrs[0], e * 0.5 + arrs[0][off(0, -1)] * 0.25)
    kb.store(arrs[-1], arrs[-1][z] * 0.5 + arrs[0][z])     # u's centre: its pending value
    return kb.build()


@pytest.mark.parametrize("rank,na,dt,shape", [
    (2, 2, "float32", (136, 45)), (2, 3, "float64", (70, 33)), (3, 2, "float32", (72, 21, 13)),
    (3, 2, "float64", (37, 18, 11)), (2, 4, "float32", (129, 40)), (2, 2, "float32", (10, 9)),
    (3, 3, "float32", (131, 17, 9)), (2, 2, "float64", (301, 27)),
])
def test_multi_array_fused_steps_match_the_oracle(rank, na, dt, shape):
    """iterate_arrays: fused steps on the multi-array TMA kernel (images of every stored
    array), then a plain launch == HALO_TRANSFER of every array + launch, K times."""
    kir = _multi_kernel(rank, na)
    k = R.CompiledKernel(kir, dt)
    assert json.loads(k.describe())["path"] == "tiled_tma_multi"
    lo, hi = [1] * rank, [1] * rank
    fields = [O.hash_field(shape, 90 + i, NP[dt]) for i in range(na)]
    hs = []
    for f in fields:
        h = R.HaloArray(shape, lo, hi, dt)
        h.set_interior(f)
        hs.append(h)
    steps = 5
    R.iterate_arrays(k, hs, steps)
    bufs = {p: O.embed(f, lo, hi, NP[dt]) for p, f in zip(kir.array_params, fields)}
    lh = {p: (lo, hi) for p in kir.array_params}
    ranges = [(1, m) for m in shape]
    for _ in range(steps):
        for b in bufs.values():
            O.halo_fill(b, lo, hi)
        O.launch(bufs, lh, kir, ranges, None, NP[dt])
    for p, h in zip(kir.array_params, hs):
        got = h.get_padded()
        assert O.equal_bits(got, bufs[p]), (p, O.first_mismatch(got, bufs[p]))
    n = launches(k)
    assert n["tiled_multi"] == steps and n["generic"] == 0, n


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_multi_array_unaligned_subranges_match_the_oracle(dt):
    """Plain launches of a multi-array kernel over sub-ranges whose x start and end fall
    inside a vector, on an odd-width interior: the multi-array TMA kernel masks its edge
    vectors; cells outside the range keep their snapshots (copy-through)."""
    kir = _multi_kernel(3, 2)
    k = R.CompiledKernel(kir, dt)
    shape = (75, 19, 11)
    lo, hi = [1] * 3, [1] * 3
    rng = np.random.default_rng(31)
    fields = [O.hash_field(shape, 120 + i, NP[dt]) for i in range(2)]
    for _ in range(5):
        ranges = []
        for m in shape:
            a = int(rng.integers(1, m // 2))
            b = int(rng.integers(a, m + 1))
            ranges.append((a, b))
        hs = []
        for f in fields:
            h = R.HaloArray(shape, lo, hi, dt)
            h.set_interior(f)
            R.halo_transfer(h)
            hs.append(h)
        R.launch(k, hs, ranges)
        bufs = {p: O.embed(f, lo, hi, NP[dt]) for p, f in zip(kir.array_params, fields)}
        for b in bufs.values():
            O.halo_fill(b, lo, hi)
        O.launch(bufs, {p: (lo, hi) for p in kir.array_params}, kir, ranges, None, NP[dt])
        for p, h in zip(kir.array_params, hs):
            got = h.get_padded()
            assert O.equal_bits(got, bufs[p]), (p, ranges, O.first_mismatch(got, bufs[p]))
    n = launches(k)
    assert n["tiled_multi"] == 5 and n["generic"] == 0, n


def test_run_pinned_batch_fp64_rank2_ragged():
    """The pipelined batch on a ragged rank-2 fp64 field (RAG tiled kernel) equals single
    runs field by field."""
    kir = stencils.box5x5()
    k = R.CompiledKernel(kir, "float64")
    shape, lo, hi = (203, 77), (2, 2), (2, 2)
    fields = [np.asfortranarray(O.hash_field(shape, 500 + i, np.float64)) for i in range(4)]
    ins = [torch.from_numpy(f.ravel(order="F").copy()).pin_memory() for f in fields]
    outs = [torch.empty_like(t).pin_memory() for t in ins]
    R.run_pinned_batch(k, shape, lo, hi, "float64", ins, outs, 3, slots=2)
    for i, f in enumerate(fields):
        want = f
        for _ in range(3):
            want = O.periodic_apply(want, kir, None, np.float64)
        got = outs[i].numpy().reshape(shape, order="F")
        assert O.equal_bits(got, want), i


@pytest.mark.parametrize("name,dt,shape,tile", [
    ("lap3d7", "float32", (512, 70, 19), (2, 8, 4, 6, 0, 1, 0, 0)),
    ("lap3d7", "float32", (301, 45, 13), (2, 8, 4, 6, 0, 1, 0, 0)),
    ("lap3d7", "float32", (512, 70, 19), (2, 8, 2, 8, 1, 1, 1, 0)),
    ("lap3d7", "float32", (301, 45, 13), (2, 8, 2, 8, 1, 1, 1, 0)),
    ("box5x5", "float64", (600, 90), (4, 4, 4, 4, 1, 1, 0, 0)),     # 4 boxes of 64+4 columns
    ("box5x5", "float64", (597, 71), (4, 4, 2, 4, 0, 1, 0, 0)),
    ("box5x5", "float64", (600, 90), (2, 8, 4, 6, 1, 1, 0, 0)),     # the tuner's two-column plan
    ("ninept2d", "float32", (1000, 77), (2, 8, 2, 8, 1, 1, 0, 0)),
])
def test_two_box_tiles_match_the_oracle(monkeypatch, name, dt, shape, tile):
    """Tiles wider than one 256-element TMA box are staged as one box per warp column
    (NB = 2 for 256-column fp32 tiles, 4 for 256-column fp64 tiles): fused steps under
    such plans (aligned and ragged x, in-band and dedicated producer, rank 2 and 3)
    equal the oracle bit for bit."""
    import ctypes
    from paper_1502_03504_b200 import _lib
    monkeypatch.setenv("LOPE_AUTOTUNE", "0")
    monkeypatch.setenv("LOPE_NO_TBLOCK", "1")
    kir = stencils.by_name(name)
    k = R.CompiledKernel(kir, dt)
    lo, hi = halos(kir)
    field = O.hash_field(shape, 77, NP[dt])
    arr = R.HaloArray(shape, lo, hi, dt)
    arr.set_interior(field)
    _lib.check(_lib.lib().lope_plan_set_variant(k.handle, ctypes.byref(arr.layout), (1 << kir.rank) - 1,
                                                (ctypes.c_int32 * 8)(*tile), 8, 0, None), "lope_plan_set_variant")
    R.iterate(k, arr, 4)
    want = O.machine_run(field, kir, 4, None, NP[dt], lo, hi)
    got = arr.get_padded()
    assert O.equal_bits(got, want), O.first_mismatch(got, want)
    n = launches(k)
    assert n["tiled"] >= 3 and n["generic"] == 0, n
