"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by gen_golden.py).

The oracle is only trusted as a checker once it reproduces, bit for bit, what
the reference ``Machine`` / ``oracle_step`` produced for the same inputs.
"""

import numpy as np
import pytest

from oracle import lope_oracle as O
from paper_1502_03504_b200 import stencils
from paper_1502_03504_b200.ir import deserialize, serialize


def test_builder_kernels_match_reference_lowering(golden_kernels):
    for name, text in golden_kernels.items():
        assert serialize(stencils.by_name(name)) == text, name


def test_serialisation_round_trips(golden_kernels, golden_random):
    meta, _ = golden_random
    for text in list(golden_kernels.values()) + [m["ir"] for m in meta]:
        assert serialize(deserialize(text)) == text


def _scal(d):
    return {k: v for k, v in d.items()}


def test_periodic_apply_matches_reference_runs(golden_runs):
    index, arr = golden_runs
    for case in index:
        kir = stencils.by_name(case["kernel"])
        ref = arr[case["tag"] + "_in"].copy()
        for _ in range(case["steps"]):
            ref = O.periodic_apply(ref, kir, _scal(case["scalars"]), np.float64)
        assert np.array_equal(ref, arr[case["tag"] + "_out"]), case["tag"]


def test_machine_run_matches_reference_runs(golden_runs):
    index, arr = golden_runs
    for case in index:
        kir = stencils.by_name(case["kernel"])
        fp = kir.footprints[kir.array_params[0]].dims
        lo = [n for n, _ in fp]
        hi = [p for _, p in fp]
        blk = O.machine_run(arr[case["tag"] + "_in"], kir, case["steps"],
                            _scal(case["scalars"]), np.float64)
        assert np.array_equal(O.interior(blk, lo, hi), arr[case["tag"] + "_out"]), case["tag"]


def test_periodic_apply_planes_equals_dense():
    kir = stencils.lap3d7()
    f = O.hash_field((10, 9, 12), 3, np.float32)
    dense = O.periodic_apply(f, kir, None, np.float32)
    part = O.periodic_apply_planes(lambda idx: f[..., idx], f.shape, kir, 0, 4, None, np.float32)
    assert O.equal_bits(part, dense[..., 0:4])
    part = O.periodic_apply_planes(lambda idx: f[..., idx], f.shape, kir, 9, 12, None, np.float32)
    assert O.equal_bits(part, dense[..., 9:12])


def test_exchange_matches_reference_blocks(golden_exchange):
    index, arr = golden_exchange
    for case in index:
        l0, h0, l1, h1 = case["widths"]
        p = case["p"]
        field = arr[case["tag"] + "_in"]
        n = field.shape[1] // p
        lo, hi = (l0, l1), (h0, h1)
        blocks = [O.embed(field[:, k * n:(k + 1) * n], lo, hi) for k in range(p)]
        O.exchange_blocks(blocks, lo, hi, axis=1)
        for k in range(p):
            assert np.array_equal(blocks[k], arr[f"{case['tag']}_blk{k + 1}"]), (case["tag"], k)


def test_random_kernels_match_reference(golden_random):
    meta, arr = golden_random
    for m in meta:
        kir = deserialize(m["ir"])
        out = O.periodic_apply(arr[f"r{m['trial']}_in"], kir, m["scalars"], np.float64)
        ref = arr[f"r{m['trial']}_out"]
        assert O.equal_bits(out, ref), m["trial"]


def test_point_source_and_layout_kats(golden_kats):
    kir = stencils.laplacian()
    f = np.zeros((4, 4)); f[1, 1] = 1.0
    got = O.periodic_apply(f, kir)
    assert np.array_equal(got, np.array(golden_kats["point_source"]))
    want = np.zeros((4, 4)); want[1, 1] = -3.0
    want[0, 1] = want[2, 1] = want[1, 0] = want[1, 2] = 1.0
    assert np.array_equal(got, want)
    f = np.zeros((4, 4)); f[0, 0] = 1.0
    assert np.array_equal(O.periodic_apply(f, kir), np.array(golden_kats["corner_source"]))
    assert golden_kats["layout_12"] == 12 and golden_kats["layout_59"] == 59


def test_subrange_and_multi_array_launch_semantics(golden_kats):
    kir = deserialize(golden_kats["subrange_ir"])
    f = np.array(golden_kats["subrange_in"])
    lo, hi = (1, 1), (1, 1)
    blk = O.embed(f, lo, hi)
    for _ in range(3):
        O.halo_fill(blk, lo, hi)
        O.launch({"u": blk}, {"u": (lo, hi)}, kir, [(2, f.shape[0] - 1), (3, f.shape[1])])
    assert np.array_equal(blk, np.array(golden_kats["subrange_out_padded"]))

    kir = deserialize(golden_kats["mix_ir"])
    f = np.array(golden_kats["mix_in"])
    u = O.embed(f, lo, hi)
    v = O.embed(f, lo, hi)
    for _ in range(4):
        O.halo_fill(u, lo, hi)
        O.halo_fill(v, lo, hi)
        O.launch({"u": u, "v": v}, {"u": (lo, hi), "v": (lo, hi)}, kir,
                 [(1, f.shape[0]), (1, f.shape[1])])
    assert np.array_equal(u, np.array(golden_kats["mix_out_u"]))
    assert np.array_equal(v, np.array(golden_kats["mix_out_v"]))


def test_fp32_restatement_is_fp32_arithmetic():
    """The fp32 oracle never promotes to fp64: outputs stay float32."""
    for name in ("heat2d", "ninept2d", "box5x5", "drift2"):
        kir = stencils.by_name(name)
        f = O.hash_field((16, 12), 7, np.float32)
        out = O.periodic_apply(f, kir, {"c": 0.25} if name == "drift2" else None, np.float32)
        assert out.dtype == np.float32


def test_hash_field_is_decomposition_independent():
    full = O.hash_field((6, 5, 8), 11, np.float32)
    planes = O.hash_planes((6, 5, 8), 11, np.arange(3, 7), np.float32)
    assert O.equal_bits(planes, full[..., 3:7])
    v = O.hash_field((1000,), 1)
    assert v.min() >= -1.0 and v.max() < 1.0 and abs(v.mean()) < 0.1


def test_periodic_apply_planes_steps_equals_dense_steps():
    """The windowed multi-step restatement (full-size sampled checks) equals K dense steps."""
    for name, shape in (("lap3d7", (12, 10, 16)), ("box5x5", (20, 24)), ("heat2d", (9, 30))):
        kir = stencils.by_name(name)
        f = O.hash_field(shape, 3, np.float64)
        want = f
        for s in range(1, 5):
            want = O.periodic_apply(want, kir, None, np.float64)
            for z0, z1 in ((0, 2), (5, 7), (shape[-1] - 2, shape[-1])):
                got = O.periodic_apply_planes_steps(lambda idx: O.hash_planes(shape, 3, idx, np.float64),
                                                    shape, kir, z0, z1, s, None, np.float64)
                assert O.equal_bits(got, want[..., z0:z1]), (name, s, z0)
