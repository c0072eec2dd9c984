"""GPU parity: liblope_b200.so kernels against the reference's golden outputs and the oracle.

fp64 runs must equal the reference ``Machine`` / ``oracle_step`` outputs bit for
bit (tests/golden, generated from the reference).  fp32 runs must equal the
fp32 restatement (oracle/lope_oracle.py) bit for bit — NaN payloads excepted
(every NaN compares equal).  All calls go through the C ABI.
"""

import json
import os

import numpy as np
import pytest

from oracle import lope_oracle as O
from paper_1502_03504_b200 import stencils
from paper_1502_03504_b200.diagnostics import RuntimeFault
from paper_1502_03504_b200.ir import deserialize

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1502_03504_b200 import runtime as R  # noqa: E402

_KCACHE = {}


def K(kir, dtype):
    key = (id(kir) if not isinstance(kir, str) else kir, dtype)
    if isinstance(kir, str):
        kir = deserialize(kir)
    name = (kir.name, kir.rank, dtype, repr(kir.body), tuple(kir.scalar_params))
    if name not in _KCACHE:
        _KCACHE[name] = R.CompiledKernel(kir, dtype)
    return _KCACHE[name]


def halos_of(kir):
    fp = kir.footprints[kir.array_params[0]].dims
    return [n for n, _ in fp], [p for _, p in fp]


def gpu_iterate(kir, field, steps, scalars, dtype, lo=None, hi=None):
    l_, h_ = halos_of(kir)
    lo = l_ if lo is None else lo
    hi = h_ if hi is None else hi
    arr = R.HaloArray(field.shape, lo, hi, dtype)
    arr.set_interior(field)
    R.iterate(K(kir, dtype), arr, steps, scalars)
    return arr


def test_fp64_matches_reference_machine_bitwise(golden_runs):
    index, arrs = golden_runs
    for case in index:
        kir = stencils.by_name(case["kernel"])
        field = arrs[case["tag"] + "_in"]
        arr = gpu_iterate(kir, field, case["steps"], case["scalars"], "float64")
        got = arr.get_interior()
        assert O.equal_bits(got, arrs[case["tag"] + "_out"]), (case["tag"], O.first_mismatch(
            got, arrs[case["tag"] + "_out"]))


def test_fp32_matches_restatement_bitwise(golden_runs):
    index, arrs = golden_runs
    for case in index:
        kir = stencils.by_name(case["kernel"])
        field = arrs[case["tag"] + "_in"].astype(np.float32)
        got = gpu_iterate(kir, field, case["steps"], case["scalars"], "float32").get_interior()
        want = field
        for _ in range(case["steps"]):
            want = O.periodic_apply(want, kir, case["scalars"], np.float32)
        assert O.equal_bits(got, want), (case["tag"], O.first_mismatch(got, want))


def test_final_halo_state_matches_reference_machine():
    """After iterate(), halo cells hold the last exchange's values, as in the reference."""
    kir = stencils.heat2d()
    field = O.hash_field((24, 20), 9, np.float64)
    arr = gpu_iterate(kir, field, 4, {}, "float64")
    want = O.machine_run(field, kir, 4, None, np.float64)
    assert O.equal_bits(arr.get_padded(), want)


def test_random_kernels_fp64_and_fp32(golden_random):
    meta, arrs = golden_random
    for m in meta:
        kir = deserialize(m["ir"])
        field = arrs[f"r{m['trial']}_in"]
        for dtype, npdt in (("float64", np.float64), ("float32", np.float32)):
            f = field.astype(npdt)
            arr = gpu_iterate(kir, f, 1, m["scalars"], dtype, lo=[2] * kir.rank, hi=[2] * kir.rank)
            got = arr.get_interior()
            if npdt == np.float64:
                want = arrs[f"r{m['trial']}_out"]
            else:
                want = O.periodic_apply(f, kir, m["scalars"], np.float32)
            # oracle_step returns a 0-d array for bodies that never read the field
            want = np.broadcast_to(want, got.shape).astype(npdt)
            assert O.equal_bits(got, want), (m["trial"], dtype, m["source"], O.first_mismatch(got, want))


def test_generic_and_tiled_paths_agree(monkeypatch):
    for name, shape, dt in (("lap3d7", (70, 37, 19), "float32"), ("box5x5", (150, 67), "float64"),
                            ("ninept2d", (131, 45), "float32"), ("drift2", (77, 41), "float32")):
        kir = stencils.by_name(name)
        f = O.hash_field(shape, 3, np.float32 if dt == "float32" else np.float64)
        sc = {"c": 0.25} if name == "drift2" else {}
        a = gpu_iterate(kir, f, 3, sc, dt).get_padded()
        monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
        b = gpu_iterate(kir, f, 3, sc, dt).get_padded()
        monkeypatch.delenv("LOPE_FORCE_GENERIC")
        assert O.equal_bits(a, b), name


def test_tile_schedule_order_invariance(monkeypatch):
    """The --shuffle-seed analogue: different CTA->unit mappings give identical bits."""
    kir = stencils.lap3d7()
    f = O.hash_field((96, 40, 33), 8, np.float32)
    base = gpu_iterate(kir, f, 2, {}, "float32").get_interior()
    for grid, zc in (("1", "16"), ("7", "5"), ("293", "1"), ("5000", "64")):
        monkeypatch.setenv("LOPE_GRID", grid)
        monkeypatch.setenv("LOPE_ZCHUNK", zc)
        got = gpu_iterate(kir, f, 2, {}, "float32").get_interior()
        assert O.equal_bits(got, base), (grid, zc)
    # banded unit walks (tile rows per band) and producer variants
    f = O.hash_field((256, 256, 20), 9, np.float32)
    monkeypatch.delenv("LOPE_GRID")
    monkeypatch.delenv("LOPE_ZCHUNK")
    base = gpu_iterate(kir, f, 2, {}, "float32").get_interior()
    for yb, zc, grid in (("2", "3", "37"), ("4", "1", "147"), ("8", "6", "100"), ("1", "2", "9")):
        monkeypatch.setenv("LOPE_YBAND", yb)
        monkeypatch.setenv("LOPE_ZCHUNK", zc)
        monkeypatch.setenv("LOPE_GRID", grid)
        got = gpu_iterate(kir, f, 2, {}, "float32").get_interior()
        assert O.equal_bits(got, base), (yb, zc, grid)


def test_halo_transfer_fills_every_padded_cell(golden_exchange):
    index, arrs = golden_exchange
    for case in index:
        if case["p"] != 1:
            continue
        l0, h0, l1, h1 = case["widths"]
        field = arrs[case["tag"] + "_in"]
        arr = R.HaloArray(field.shape, (l0, l1), (h0, h1), "float64")
        arr.set_interior(field)
        R.halo_transfer(arr)
        assert np.array_equal(arr.get_padded(), arrs[case["tag"] + "_blk1"]), case["tag"]


def test_subrange_launch_copies_through(golden_kats):
    kir = deserialize(golden_kats["subrange_ir"])
    f = np.array(golden_kats["subrange_in"])
    arr = R.HaloArray(f.shape, (1, 1), (1, 1), "float64")
    arr.set_interior(f)
    k = K(kir, "float64")
    for _ in range(3):
        R.halo_transfer(arr)
        R.launch(k, [arr], [(2, f.shape[0] - 1), (3, f.shape[1])])
    assert np.array_equal(arr.get_padded(), np.array(golden_kats["subrange_out_padded"]))


def test_two_array_kernel_and_pending_centre(golden_kats):
    kir = deserialize(golden_kats["mix_ir"])
    f = np.array(golden_kats["mix_in"])
    u = R.HaloArray(f.shape, (1, 1), (1, 1), "float64", name="u")
    v = R.HaloArray(f.shape, (1, 1), (1, 1), "float64", name="v")
    u.set_interior(f)
    v.set_interior(f)
    k = K(kir, "float64")
    for _ in range(4):
        R.halo_transfer(u)
        R.halo_transfer(v)
        R.launch(k, [u, v])
    assert np.array_equal(u.get_padded(), np.array(golden_kats["mix_out_u"]))
    assert np.array_equal(v.get_padded(), np.array(golden_kats["mix_out_v"]))
    twice = deserialize(golden_kats["twice_ir"])
    g = np.full((4, 4), 1.5)
    arr = R.HaloArray(g.shape, (1, 1), (1, 1), "float64")
    arr.set_interior(g)
    R.launch(K(twice, "float64"), [arr])
    assert np.array_equal(arr.get_interior(), g * 2 + 1)


def test_point_source_and_fixed_point_kats(golden_kats):
    kir = stencils.laplacian()
    f = np.zeros((4, 4)); f[1, 1] = 1.0
    assert np.array_equal(R.run(kir, f, 1, dtype="float64"), np.array(golden_kats["point_source"]))
    f = np.zeros((4, 4)); f[0, 0] = 1.0
    assert np.array_equal(R.run(kir, f, 1, dtype="float64"), np.array(golden_kats["corner_source"]))
    ones = np.full((8, 8), 1.0)
    assert np.array_equal(R.run(kir, ones, 25, dtype="float64"), ones)


def test_empty_range_and_faults():
    kir = stencils.heat2d()
    f = O.hash_field((8, 8), 1, np.float64)
    arr = R.HaloArray(f.shape, (1, 1), (1, 1), "float64")
    arr.set_interior(f)
    k = K(kir, "float64")
    R.launch(k, [arr], [(1, 0), (1, 8)])
    assert np.array_equal(arr.get_interior(), f)
    with pytest.raises(RuntimeFault) as e:
        R.launch(k, [arr], [(1, 9), (1, 8)])
    assert e.value.code == "E108"
    for rng in ([(0, -1), (1, 8)], [(1, 8), (3, 9)], [(20, 10), (1, 8)]):   # empty but out of bounds
        with pytest.raises(RuntimeFault) as e:
            R.launch(k, [arr], rng)
        assert e.value.code == "E108", rng
    thin = R.HaloArray((8, 8), (0, 1), (1, 1), "float64")
    with pytest.raises(RuntimeFault) as e:
        R.launch(k, [thin])
    assert e.value.code == "E102"
    narrow = R.HaloArray((1, 8), (2, 1), (2, 1), "float64")      # halo wider than interior (F8)
    with pytest.raises(RuntimeFault) as e:
        R.halo_transfer(narrow)
    assert e.value.code == "E108"


def test_device_hash_fill_matches_oracle():
    for dt, npdt in (("float32", np.float32), ("float64", np.float64)):
        arr = R.HaloArray((33, 17, 9), (1, 1, 1), (1, 1, 1), dt)
        arr.fill_hash(1234)
        assert O.equal_bits(arr.get_interior(), O.hash_field((33, 17, 9), 1234, npdt))
        arr = R.HaloArray((20, 12), (2, 2), (2, 2), dt)
        arr.fill_hash(77, global_extent=(20, 48), global_origin=(0, 24))
        assert O.equal_bits(arr.get_interior(), O.hash_field((20, 48), 77, npdt)[:, 24:36])


def _planes_check(arr, kir, gshape, seed, npdt, planes, steps_done=1):
    assert steps_done == 1
    L = arr.layout
    v = arr.interior_view()            # [c2, c1, c0]
    for z0, z1 in planes:
        got = v[z0:z1].cpu().numpy().transpose(2, 1, 0) if arr.rank == 3 else None
        if arr.rank == 2:
            got = v[0, z0:z1, :].cpu().numpy().transpose(1, 0)
        want = O.periodic_apply_planes(lambda idx: O.hash_planes(gshape, seed, idx, npdt), gshape,
                                       kir, z0, z1, None, npdt)
        assert O.equal_bits(got, want), (z0, z1, O.first_mismatch(got, want))


@pytest.mark.parametrize("name,shape,dt", [
    ("lap3d7", (1024, 1024, 1024), "float32"),
    ("ninept2d", (16384, 16384), "float32"),
    ("box5x5", (32768, 32768), "float64"),
])
def test_full_size_one_step_sampled_planes(name, shape, dt):
    """BASELINE sizes: device-generated input, one step, sampled planes vs the oracle."""
    kir = stencils.by_name(name)
    npdt = np.float32 if dt == "float32" else np.float64
    lo, hi = halos_of(kir)
    arr = R.HaloArray(shape, lo, hi, dt)
    arr.fill_hash(20260823)
    R.iterate(K(kir, dt), arr, 1)
    n = shape[-1]
    _planes_check(arr, kir, shape, 20260823, npdt, [(0, 2), (n // 2 - 1, n // 2 + 1), (n - 2, n)])
    del arr
    torch.cuda.empty_cache()


def test_full_size_multi_step_tiled_equals_generic(monkeypatch):
    """Config 3 at full size, 5 steps: TMA tiled path == independent generic path, bit for bit."""
    kir = stencils.lap3d7()
    shape = (1024, 1024, 1024)
    a = R.HaloArray(shape, (1, 1, 1), (1, 1, 1), "float32")
    a.fill_hash(5)
    R.iterate(K(kir, "float32"), a, 5)
    monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
    b = R.HaloArray(shape, (1, 1, 1), (1, 1, 1), "float32")
    b.fill_hash(5)
    R.iterate(K(kir, "float32"), b, 5)
    assert torch.equal(a.padded_view().contiguous().view(torch.int32),
                       b.padded_view().contiguous().view(torch.int32))
    del a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,shape,dt", [("lap3d7", (256, 96, 64), "float32"),
                                           ("ninept2d", (512, 256), "float32"),
                                           ("box5x5", (256, 128), "float64")])
def test_plan_tuning_is_bitwise_transparent(name, shape, dt):
    """The online tuner runs real steps under every candidate plan and keeps one;
    the field after tuning plus further steps equals the plain run of as many steps."""
    import json
    kir = stencils.by_name(name)
    npdt = np.float32 if dt == "float32" else np.float64
    field = O.hash_field(shape, 23, npdt)
    k = R.CompiledKernel(kir, dt)
    l_, h_ = halos_of(kir)
    arr = R.HaloArray(shape, l_, h_, dt)
    arr.set_interior(field)
    R.halo_transfer(arr)
    rep = k.tune(arr)
    t = k._tuners[next(iter(k._tuners))]
    n_tune = t.steps_needed if len(t.cands) > 1 else 0
    assert rep["best"] is not None or len(t.cands) <= 1
    if len(t.cands) > 1:
        assert len(json.loads(k.describe())["plans"]) == 1
    R.step(k, arr)
    R.launch(k, [arr])
    plain = gpu_iterate(kir, field, n_tune + 2, {}, dt).get_interior()
    assert O.equal_bits(arr.get_interior(), plain)


@pytest.mark.parametrize("name,shape,dt,n", [("heat2d", (1024, 1024), "float32", 17),
                                             ("heat2d", (300, 170), "float64", 17),
                                             ("box5x5", (256, 192), "float64", 8),
                                             ("drift2", (288, 160), "float32", 16),
                                             ("ninept2d", (272, 44), "float32", 17),
                                             ("box5x5", (288, 64), "float32", 12),
                                             ("heat2d", (100, 60), "float32", 6),
                                             ("heat2d", (1000, 333), "float32", 16)])
def test_temporal_blocking_is_bitwise_identical(monkeypatch, name, shape, dt, n):
    """multi_step (4 steps per launch in shared memory for rank 2) leaves the same
    padded block -- interior and periodic halo images -- as n single fused steps."""
    kir = stencils.by_name(name)
    npdt = np.float32 if dt == "float32" else np.float64
    sc = {"c": 0.25} if name == "drift2" else None
    field = O.hash_field(shape, 29, npdt)
    l_, h_ = halos_of(kir)
    k = K(kir, dt)
    a = R.HaloArray(shape, l_, h_, dt)
    a.set_interior(field)
    R.halo_transfer(a)
    R.multi_step(k, a, n, sc)
    b = R.HaloArray(shape, l_, h_, dt)
    b.set_interior(field)
    R.halo_transfer(b)
    for _ in range(n):
        R.step(k, b, sc)
    assert O.equal_bits(a.get_padded(), b.get_padded()), O.first_mismatch(a.get_padded(), b.get_padded())
    want = field
    for _ in range(n):
        want = O.periodic_apply(want, kir, sc, npdt)
    assert O.equal_bits(a.get_interior(), want)


def test_step_graph_with_temporal_blocking_matches_single_steps():
    kir = stencils.heat2d()
    field = O.hash_field((512, 256), 31, np.float32)
    k = K(kir, "float32")
    a = R.HaloArray(field.shape, [1, 1], [1, 1], "float32")
    a.set_interior(field)
    R.halo_transfer(a)
    g = R.StepGraph(k, a, 16)          # construction leaves the field alone
    assert O.equal_bits(a.get_interior(), field)
    g.replay()
    torch.cuda.synchronize()
    assert g.launches < 16
    want = field
    for _ in range(16):
        want = O.periodic_apply(want, kir, None, np.float32)
    assert O.equal_bits(a.get_interior(), want)


def test_full_size_every_plan_family_matches_generic(monkeypatch):
    """Config 3 at full size: each execution-plan family the tuner can pick (in-band
    producer with long z-chunks, dedicated producer with short chunks, deeper rings)
    gives the generic kernel's bits after 3 steps."""
    monkeypatch.setenv("LOPE_AUTOTUNE", "0")
    kir = stencils.lap3d7()
    shape = (1024, 1024, 1024)
    monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
    ref = R.HaloArray(shape, (1, 1, 1), (1, 1, 1), "float32")
    ref.fill_hash(11)
    R.iterate(K(kir, "float32"), ref, 3)
    want = ref.padded_view().contiguous().view(torch.int32).clone()
    del ref
    monkeypatch.delenv("LOPE_FORCE_GENERIC")
    k = R.CompiledKernel(kir, "float32")
    a = R.HaloArray(shape, (1, 1, 1), (1, 1, 1), "float32")
    t = R.PlanTuner(k, a.layout, 7)
    assert len(t.cands) >= 6
    for cand in t.cands[::4]:
        t._set(*cand)
        a.fill_hash(11)
        R.iterate(k, a, 3)
        got = a.padded_view().contiguous().view(torch.int32)
        assert torch.equal(got, want), cand
    del a
    torch.cuda.empty_cache()


def test_random_kernels_tiled_vs_generic_on_ragged_shapes(monkeypatch, golden_random):
    """Every golden random kernel of rank 2/3 on ragged shapes (x not a multiple of the
    tile, odd y and z), asymmetric halos wider than the footprint, fp32 and fp64, three
    fused steps plus a final launch: the TMA-tiled path (every plan family the tuner can
    pick) equals the generic path bit for bit, padded block included."""
    meta, _ = golden_random
    rng = np.random.default_rng(2024)
    monkeypatch.setenv("LOPE_AUTOTUNE", "0")
    checked = 0
    for m in meta:
        kir = deserialize(m["ir"])
        if kir.rank < 2 or len(kir.array_params) != 1:
            continue
        fp = kir.footprints[kir.array_params[0]].dims
        lo = [int(n) + int(rng.integers(0, 2)) for n, _ in fp]
        hi = [int(p) + int(rng.integers(0, 2)) for _, p in fp]
        for dt, npdt in (("float32", np.float32), ("float64", np.float64)):
            vx = 4 if dt == "float32" else 2
            mx = int(rng.integers(9, 50)) * vx
            shape = (mx, int(rng.integers(11, 71))) + ((int(rng.integers(5, 23)),) if kir.rank == 3 else ())
            if any(s < l + h for s, l, h in zip(shape, lo, hi)):
                continue
            field = O.hash_field(shape, int(m["trial"]) + 7, npdt)
            k = R.CompiledKernel(kir, dt)
            outs = []
            for generic in (False, True):
                if generic:
                    monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
                a = R.HaloArray(shape, lo, hi, dt)
                a.set_interior(field)
                R.iterate(k, a, 4, m["scalars"])
                outs.append(a.get_padded())
                monkeypatch.delenv("LOPE_FORCE_GENERIC", raising=False)
            assert O.equal_bits(outs[0], outs[1]), (m["trial"], dt, shape, lo, hi, m["source"])
            if kir.rank == 3 and dt == "float32":
                t = R.PlanTuner(k, R.HaloArray(shape, lo, hi, dt).layout, 7)
                for cand in t.cands[::3]:
                    t._set(*cand)
                    a = R.HaloArray(shape, lo, hi, dt)
                    a.set_interior(field)
                    R.iterate(k, a, 4, m["scalars"])
                    assert O.equal_bits(a.get_padded(), outs[1]), (m["trial"], cand, shape)
            checked += 1
    assert checked >= 40


@pytest.mark.parametrize("rank,na,dt", [(2, 2, "float32"), (2, 3, "float64"), (3, 2, "float32"),
                                         (3, 2, "float64"), (2, 4, "float32")])
def test_multi_array_tiled_equals_generic(monkeypatch, rank, na, dt):
    """Kernels over 2-4 arrays run on the multi-array TMA kernel (one box per array per
    plane); full and sub-range launches equal the generic kernel bit for bit (padded
    blocks included); tools/fuzz_gpu.py checks two-array kernels against the oracle."""
    import json
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder(f"multi{rank}{na}", rank)
    arrs = [kb.array(n) for n in "uvwx"[:na]]
    z = (0,) * rank

    def off(d, s_):
        o = [0] * rank
        o[d] = s_
        return tuple(o)

    e = arrs[0][z]
    for i, a in enumerate(arrs[1:], 1):
        e = e + (a[off(0, 1)] - a[off(rank - 1, -1)]) * (0.25 * i) + a[off(1, -1)] / 3.0
    kb.store(arrs[0], e)
    kb.store(arrs[-1], arrs[-1][z] * 0.5 + arrs[0][z])
    kir = kb.build()
    k = K(kir, dt)
    assert json.loads(k.describe())["path"] == "tiled_tma_multi"
    npdt = np.float32 if dt == "float32" else np.float64
    shape = (136, 45) if rank == 2 else (72, 21, 13)
    fields = [O.hash_field(shape, 60 + i, npdt) for i in range(na)]
    lo, hi = [1] * rank, [1] * rank
    outs = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
        hs = []
        for f in fields:
            h = R.HaloArray(shape, lo, hi, dt)
            h.set_interior(f)
            R.halo_transfer(h)
            hs.append(h)
        R.launch(k, hs)
        sub = [(5, shape[0] - 3), (2, shape[1] - 1)] + ([(2, shape[2])] if rank == 3 else [])
        for h in hs:
            R.halo_transfer(h)
        R.launch(k, hs, sub)
        outs.append([h.get_padded() for h in hs])
        monkeypatch.delenv("LOPE_FORCE_GENERIC", raising=False)
        if not generic:   # the multi-array kernel itself ran (no silent generic fallback)
            n = json.loads(k.describe())["launches"]
            assert n["tiled_multi"] == 2 and n["generic"] == 0, n
    for a_, b_ in zip(*outs):
        assert O.equal_bits(a_, b_)


def test_run_pinned_on_a_side_stream_with_the_default_stream_busy():
    """buffers used on a caller's stream are zero-filled on that stream, so a
    busy default stream cannot delay a fill past the upload or the first step's stores."""
    kir = stencils.heat2d()
    shape = (512, 384)
    field = O.hash_field(shape, 41, np.float32)
    host_in = torch.from_numpy(np.asfortranarray(field).ravel(order="K").copy()).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    side = torch.cuda.Stream()
    k = K(kir, "float32")
    torch.cuda._sleep(200_000_000)               # ~0.1 s of work queued on the default stream
    R.run_pinned(k, shape, (1, 1), (1, 1), "float32", host_in, host_out, 9, stream=side)
    got = host_out.numpy().reshape(shape, order="F")
    want = field
    for _ in range(9):
        want = O.periodic_apply(want, kir, None, np.float32)
    assert O.equal_bits(got, want)
    torch.cuda.synchronize()


def test_run_pinned_batch_matches_single_runs():
    """run_pinned_batch (uploads, iterations and downloads of independent fields on three
    streams, device slots reused) gives every field the bits run_pinned gives it."""
    kir = stencils.lap3d7()
    k = K(kir, "float32")
    shape, lo, hi = (136, 40, 23), (1, 1, 1), (1, 1, 1)
    fields = [np.asfortranarray(O.hash_field(shape, 300 + i, np.float32)) for i in range(5)]
    ins = [torch.from_numpy(f.ravel(order="F").copy()).pin_memory() for f in fields]
    outs = [torch.empty_like(t).pin_memory() for t in ins]
    R.run_pinned_batch(k, shape, lo, hi, "float32", ins, outs, 4, slots=3)
    for i, t in enumerate(ins):
        ref = torch.empty_like(t).pin_memory()
        R.run_pinned(k, shape, lo, hi, "float32", t, ref, 4)
        assert torch.equal(outs[i].view(torch.int32), ref.view(torch.int32)), i
        want = fields[i]
        for _ in range(4):
            want = O.periodic_apply(want, kir, None, np.float32)
        got = outs[i].numpy().reshape(shape, order="F")
        assert O.equal_bits(got, want), i
