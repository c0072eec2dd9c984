"""CPU-side checks of the C ABI: the library loads, exports every symbol the header
declares, lays out blocks as the reference does, compiles kernels (NVRTC needs no
GPU) and rejects bad input with the reference's error codes.  No kernel runs here."""

import json
import re

import pytest

from conftest import REPO
from paper_1502_03504_b200 import _lib, stencils
from paper_1502_03504_b200.diagnostics import RuntimeFault
from paper_1502_03504_b200.ir import KernelBuilder, serialize


def header_symbols():
    text = (REPO / "include" / "lope_b200.h").read_text()
    return sorted(set(re.findall(r"\b(lope_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.lope_abi_version() == 1


def test_layout_matches_reference_storage_layout():
    # StorageLayout((8,4,3),(1,2,0),(1,0,1)): padded (10,6,4) (tests/test_layout.py:24-29)
    L = _lib.make_layout(3, "f32", (8, 4, 3), (1, 2, 0), (1, 0, 1))
    assert tuple(L.padded) == (10, 6, 4)
    # column-major like the reference, each row shifted so the interior starts on a
    # 64-byte atom with an atom of room for each halo side, pitch in whole atoms
    assert L.base == 16 - 1 and (L.base + L.lo[0]) % 16 == 0
    assert L.stride[0] == 1 and L.stride[1] == 48 and L.stride[2] == 48 * 6
    assert L.count == 48 * 6 * 4
    # frozen KAT (test_layout.py:14-21): 8x4 interior, halo 1, centre (1,1)+(1,0) -> padded (2,1);
    # the reference's linear index 12 = 2 + 1*10 becomes base + 2 + 1*stride here
    L2 = _lib.make_layout(2, "f64", (8, 4), (1, 1), (1, 1))
    assert L2.stride[1] == 24 and L2.base == 7
    ref_linear = lambda c0, c1: c0 + c1 * 10
    dev_linear = lambda c0, c1: L2.base + c0 + c1 * L2.stride[1]
    assert ref_linear(2, 1) == 12 and ref_linear(9, 5) == 59
    assert dev_linear(2, 1) == 7 + 2 + 24 and dev_linear(9, 5) == 7 + 9 + 5 * 24


def test_layout_rejects_bad_shapes():
    with pytest.raises(RuntimeFault) as e:
        _lib.make_layout(2, "f32", (0, 4), (1, 1), (1, 1))
    assert e.value.code == "E108"
    with pytest.raises(RuntimeFault) as e:
        _lib.make_layout(2, "f32", (4, 4), (9, 1), (1, 1))
    assert e.value.code == "E108"


def test_face_spans_are_contiguous_planes():
    L = _lib.make_layout(3, "f32", (8, 6, 10), (1, 1, 2), (1, 1, 1))
    plane = L.stride[2]
    assert _lib.face_span(L, 0) == (0, 2 * plane)
    assert _lib.face_span(L, 1) == ((2 + 10) * plane, 1 * plane)
    assert _lib.face_span(L, 2) == (2 * plane, 1 * plane)
    assert _lib.face_span(L, 3) == (10 * plane, 2 * plane)


def test_kernels_compile_and_describe():
    for name in ("lap3d7", "ninept2d", "box5x5", "drift2", "avg3"):
        h = _lib.compile_kernel(serialize(stencils.by_name(name)), "f32")
        d = json.loads(_lib.describe(h))
        assert d["name"] == name
        if name in ("lap3d7", "ninept2d", "box5x5", "drift2"):
            assert d["path"] == "tiled_tma"
        else:
            assert d["path"] == "row"       # rank 1: the vector row kernel
            assert "lope_row(" in _lib.source(h)
        assert set(d["launches"]) == {"tiled", "tiled_multi", "row", "tblock", "generic"}
        src = _lib.source(h)
        assert "__fadd_rn" in src and "cp.async.bulk.tensor" in src
        _lib.destroy_kernel(h)


def test_prepared_variants_are_the_tuner_candidates():
    """lope_kernel_prepare compiles the plan tuner's tile variants (NVRTC, no GPU):
    every one fits shared memory, the 3-D fp32 list is the six variants behind the
    nine 3-D plans, and wide-footprint fp64 2-D kernels get the two-warp-column plan."""
    def variants(name, dt):
        h = _lib.compile_kernel(serialize(stencils.by_name(name)), dt)
        try:
            _lib.check(_lib.lib().lope_kernel_prepare(h), "lope_kernel_prepare")
            return json.loads(_lib.describe(h))["variants"]
        finally:
            _lib.destroy_kernel(h)

    v3 = variants("lap3d7", "f32")
    assert all(v["tiled"] for v in v3)
    assert [(v["tile"], v["producer_warp"], v["shfl"], v["nb"]) for v in v3] == [
        ([1, 16, 2, 8], 0, 0, 0), ([1, 16, 2, 8], 0, 0, 1), ([1, 16, 2, 8], 1, 1, 0),
        ([1, 16, 2, 10], 1, 1, 0), ([1, 16, 2, 12], 1, 1, 0), ([1, 8, 4, 8], 0, 0, 0)]
    v5 = variants("box5x5", "f64")
    assert all(v["tiled"] for v in v5)
    assert {"tile": [2, 8, 4, 6], "producer_warp": 1, "shfl": 0, "nb": 0, "rag": 0, "tiled": True} in v5
    assert all(v["tile"][0] == 1 for v in variants("heat2d", "f32"))


def test_constants_cross_the_boundary_exactly():
    k = KernelBuilder("c", 2)
    u = k.array("u")
    k.store(u, u[0, 0] * 0.1 + 1e-300)
    h = _lib.compile_kernel(serialize(k.build()), "f64")
    src = _lib.source(h)
    assert "T(" + (0.1).hex().replace("0x1.", "0x1.") in src or "0x1.999999999999ap-4" in src
    _lib.destroy_kernel(h)


def test_bad_ir_is_rejected():
    with pytest.raises(RuntimeFault) as e:
        _lib.compile_kernel("LOPE1\nkernel k 2\narray u\nstore u r v 0 0\nend\n", "f32")
    assert e.value.code == "E104"
    with pytest.raises(RuntimeFault):
        _lib.compile_kernel("LOPE1\nkernel k 2\narray u\nstore u r u 0 0\nstore u r u 1 0\nend\n", "f32")


def test_compiled_kernel_object_without_gpu():
    from paper_1502_03504_b200.runtime import CompiledKernel
    for dt in ("float32", "float64", _lib.F32):
        k = CompiledKernel(stencils.drift2(), dt)
        d = json.loads(k.describe())
        assert d["scalars"] == [["c", "real"]] and d["footprints"] == [[[2, 0], [1, 1]]]
        rs, is_ = k.scalar_args({"c": 0.25})
        assert rs[0] == 0.25
    with pytest.raises(RuntimeFault):
        k.scalar_args({})


def test_machine_dropin_subclasses_the_reference_machine():
    from conftest import import_lopec
    if not import_lopec(allow_reference_tree=True):
        pytest.skip("lopec not importable")
    import lopec.runtime
    from paper_1502_03504_b200.machine import machine_class
    cls = machine_class()
    assert issubclass(cls, lopec.runtime.Machine)
    for name in ("_launch", "_halo_exchange", "gather", "run"):
        assert getattr(cls, name) is not getattr(lopec.runtime.Machine, name), name


def test_header_is_plain_c_and_the_c_driver_links(tmp_path):
    """include/lope_b200.h compiles as C99 (no C++ or torch types in the boundary) and
    tools/abi_bench.c -- a host that binds only the C ABI -- links against the library."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    cuda_inc = "/usr/local/cuda/include"
    src = tmp_path / "use.c"
    src.write_text('#include "lope_b200.h"\nint main(void) { return lope_abi_version() == 1 ? 0 : 1; }\n')
    r = subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-fsyntax-only", f"-I{REPO / 'include'}",
                        f"-I{cuda_inc}", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = tmp_path / "abi_bench"
    r = subprocess.run([gcc, "-O2", "-o", str(out), str(REPO / "tools" / "abi_bench.c"), f"-I{REPO / 'include'}",
                        f"-I{cuda_inc}", f"-L{REPO / 'paper_1502_03504_b200'}", "-llope_b200",
                        "-L/usr/local/cuda/lib64", "-lcudart"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_plan_watchdog_falls_back_only_on_the_slow_mode():
    """PlanTuner's watchdog (CPU logic): a window of steps >= SLOW x the fast-mode time
    switches to the long-chunk plan; power-cap-sized slowdowns do not."""
    from paper_1502_03504_b200.runtime import PlanTuner
    t = PlanTuner.__new__(PlanTuner)
    t.cands = [(0, 64, 0), (2, 6, 0)]
    t.report = {"fallback": None}
    t._watch = []
    calls = []
    t._set = lambda *c: calls.append(c)
    # fast mode 1.40 ms, power cap pushes steps to 1.52 ms: keep the plan
    t._safe, t._safe_ms, t.monitoring, t._durations = (0, 1.40), 1.62, True, [1.52] * PlanTuner.WATCH
    t._check_window()
    assert t.monitoring and not calls and t.report["fallback"] is None
    # slow mode (1.80 ms) but the long-chunk plan tuned at 1.78 ms: switching gains nothing
    t._safe_ms = 1.78
    t._durations = [1.80] * PlanTuner.WATCH
    t._check_window()
    assert t.monitoring and not calls and t.report["fallback"] is None
    # slow mode (1.95 ms): fall back to the long-chunk candidate 0
    t._durations = [1.95] * PlanTuner.WATCH
    t._check_window()
    assert not t.monitoring and calls == [(0, 64, 0)]
    assert t.report["fallback"]["to"] == [0, 64, 0]


def test_boundary_rejects_bad_calls_with_reference_codes():
    """Argument checks of the C ABI run before any device work (so they are testable on
    the CPU) and come back as the reference's E-codes."""
    import ctypes
    L = _lib.lib()
    h = _lib.compile_kernel(serialize(stencils.lap3d7()), "f32")
    lay = _lib.make_layout(3, "f32", (64, 32, 16), (1, 1, 1), (1, 1, 1))
    thin = _lib.make_layout(3, "f32", (64, 32, 16), (0, 1, 1), (1, 1, 1))
    lay64 = _lib.make_layout(3, "f64", (64, 32, 16), (1, 1, 1), (1, 1, 1))
    rs, is_ = (ctypes.c_double * 1)(), (ctypes.c_int64 * 1)()
    A, B = ctypes.c_void_p(0x1000), ctypes.c_void_p(0x2000)

    assert L.lope_step(h, ctypes.byref(lay), A, A, rs, is_, 7, None) == 108            # in == out
    assert L.lope_step(h, ctypes.byref(thin), A, B, rs, is_, 7, None) == 102           # footprint > halo
    assert L.lope_step(h, ctypes.byref(lay64), A, B, rs, is_, 7, None) == 108          # dtype mismatch
    assert L.lope_step(h, ctypes.byref(lay), None, B, rs, is_, 7, None) == 202         # unallocated
    assert L.lope_step_planes(h, ctypes.byref(lay), A, B, 3, 40, rs, is_, 7, None) == 108   # plane range
    live = ctypes.c_int32()
    assert L.lope_step_multi(h, ctypes.byref(lay), A, B, -1, rs, is_, None, ctypes.byref(live)) == 108
    box = (ctypes.c_int64 * 3)(60, 0, 0)
    ext = (ctypes.c_int64 * 3)(10, 1, 1)
    assert L.lope_box_pack(ctypes.byref(lay), A, box, ext, B, None) == 108               # box leaves block
    assert L.lope_copy_box(ctypes.byref(lay), A, B, box, box, ext, None) == 108
    ptrs = (ctypes.c_void_p * 2)(A, B)
    boxes = (ctypes.c_int64 * 6)(0, 0, 0, 60, 0, 0)
    exts = (ctypes.c_int64 * 6)(1, 1, 1, 10, 1, 1)
    assert L.lope_copy_boxes(ctypes.byref(lay), 2, ptrs, ptrs, boxes, boxes, exts, None) == 108   # 2nd box leaves
    assert L.lope_copy_boxes(ctypes.byref(lay), -1, ptrs, ptrs, boxes, boxes, exts, None) == 108
    nulls = (ctypes.c_void_p * 2)(A, None)
    assert L.lope_copy_boxes(ctypes.byref(lay), 2, nulls, ptrs, boxes, boxes, exts, None) == 202
    assert L.lope_copy_boxes(ctypes.byref(lay), 0, None, None, None, None, None, None) == 0
    assert L.lope_plan_set(h, ctypes.byref(lay), 7, 99, 4, 0) == 108                     # no such variant
    assert L.lope_ipc_close(ctypes.c_void_p(0x1234)) == 108                               # never opened
    # lope_launch bounds-checks every dim before an empty range returns (runtime.py:583-595)
    ins = (ctypes.c_void_p * 1)(A)
    outs = (ctypes.c_void_p * 1)(B)
    for rng in ((0, -1, 1, 32, 1, 16), (1, 64, 1, 32, 20, 17), (1, 64, 5, 3, 1, 17)):
        assert L.lope_launch(h, ctypes.byref(lay), (ctypes.c_int64 * 6)(*rng), ins, outs, rs, is_, None) == 108, rng
    assert b"" != L.lope_last_error()
    _lib.destroy_kernel(h)


def test_step_arrays_rejects_bad_calls_with_reference_codes():
    """lope_step_arrays (fused steps of multi-array kernels) checks its arguments before
    any device work: aliasing outputs and layout mismatches are E108, a footprint wider
    than an array's halo E102, a missing buffer E202."""
    import ctypes
    L = _lib.lib()
    kb = KernelBuilder("two", 2)
    u, v = kb.array("u"), kb.array("v")
    kb.store(u, u[0, 0] + 0.5 * (v[1, 0] + v[0, -1]))
    h = _lib.compile_kernel(serialize(kb.build()), "f32")
    lay = _lib.make_layout(2, "f32", (64, 32), (1, 1), (1, 1))
    other = _lib.make_layout(2, "f32", (64, 16), (1, 1), (1, 1))
    thin = _lib.make_layout(2, "f32", (64, 32), (0, 0), (0, 1))
    rs, is_ = (ctypes.c_double * 1)(), (ctypes.c_int64 * 1)()
    A, B, C = 0x1000, 0x2000, 0x3000

    def call(layouts, ins, outs):
        lays = (_lib.Layout * 2)(*layouts)
        return L.lope_step_arrays(h, lays, (ctypes.c_void_p * 2)(*ins), (ctypes.c_void_p * 2)(*outs),
                                  rs, is_, 3, None)

    assert call((lay, lay), (A, B), (A, None)) == 108          # u's output aliases its snapshot
    assert call((lay, other), (A, B), (C, None)) == 108        # different interiors
    assert call((lay, thin), (A, B), (C, None)) == 102         # v read at x+1 / y-1, halo (0,0)/(0,1)
    assert call((lay, lay), (A, None), (C, None)) == 202       # v not allocated
    assert call((lay, lay), (A, B), (None, None)) == 202       # stored u has no output
    _lib.destroy_kernel(h)


def test_comm_boundary_checks_without_a_gpu():
    """lope_comm's argument and setup-order checks (no device work): the reference's
    E-codes for a bad image index (E201) and missing setup (E202)."""
    import ctypes
    L = _lib.lib()
    h = ctypes.c_void_p()
    assert L.lope_comm_create(0, 0, ctypes.byref(h)) == 201
    assert L.lope_comm_create(4, 4, ctypes.byref(h)) == 201
    assert L.lope_comm_create(4, -1, ctypes.byref(h)) == 201
    assert L.lope_comm_create(4, 1, ctypes.byref(h)) == 0 and h.value
    assert L.lope_comm_record_size() >= 256
    recs = ctypes.create_string_buffer(4 * L.lope_comm_record_size())
    assert L.lope_comm_connect(h, recs) == 202                      # export first
    assert L.lope_halo_exchange(h, 0, 7, None) == 202
    assert L.lope_comm_step(h, ctypes.c_void_p(0x10), 0, None, None, None) == 202
    lay = _lib.make_layout(3, "f32", (64, 32, 16), (1, 1, 1), (1, 1, 1))
    assert L.lope_comm_export(h, ctypes.byref(lay), None, None, recs) == 202
    A = ctypes.c_void_p(0x1000)
    assert L.lope_comm_export(h, ctypes.byref(lay), A, A, recs) == 108   # same buffer twice
    thin = _lib.make_layout(3, "f32", (64, 32, 1), (1, 1, 2), (1, 1, 2))
    assert L.lope_comm_export(h, ctypes.byref(thin), A, ctypes.c_void_p(0x2000), recs) == 108   # F8
    r, n, e, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint32(), ctypes.c_int32()
    assert L.lope_comm_info(h, ctypes.byref(r), ctypes.byref(n), ctypes.byref(e), ctypes.byref(t)) == 0
    assert (r.value, n.value, e.value, t.value) == (1, 4, 0, 0)
    assert L.lope_halo_exchange_end(h, None) == 0                   # nothing pending
    assert L.lope_comm_destroy(h) == 0


def _sass_opcodes(kir, dt):
    """NVRTC-compile (no GPU) into a scratch cache and list the tiled kernels' SASS opcodes."""
    import collections
    import pathlib
    import shutil
    import subprocess
    import tempfile
    if shutil.which("cuobjdump") is None and not pathlib.Path("/usr/local/cuda/bin/cuobjdump").exists():
        pytest.skip("cuobjdump not available")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    tmp = tempfile.mkdtemp()
    try:
        _lib.lib().lope_set_cache_dir(tmp.encode())
        h = _lib.compile_kernel(serialize(kir), dt)
        _lib.destroy_kernel(h)
        ops = collections.Counter()
        for f in pathlib.Path(tmp).glob("*.cubin"):
            for fun in ("lope_tiled", "lope_tiled_multi", "lope_tblock", "lope_row"):
                out = subprocess.run([exe, "-sass", "-fun", fun, str(f)], capture_output=True, text=True).stdout
                for m in re.finditer(r"/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", out):
                    ops[m.group(2)] += 1
        return ops
    finally:
        _lib.lib().lope_set_cache_dir(str(_lib.CACHE_DIR).encode())
        shutil.rmtree(tmp, ignore_errors=True)


@pytest.mark.parametrize("name", ["lap3d7", "heat2d", "ninept2d", "laplacian", "drift2"])
def test_no_contraction_in_kernels_without_division(name):
    """The parity contract forbids fusing a product into a following add (numpy rounds
    each node).  fp32 bodies evaluate point pairs with FADD2 / FMUL2; ptxas would fuse
    a paired multiply into FFMA2, so products stay scalar.  Kernels without a division
    (whose exact reciprocal step uses FMA on purpose) must contain no FFMA / FFMA2 / DFMA
    at all; the temporal-blocking kernel does pair."""
    kir = stencils.by_name(name)
    for dt in ("f32", "f64"):
        ops = _sass_opcodes(kir, dt)
        assert sum(ops.values()) > 100, ops
        for op in ("FFMA", "FFMA2", "DFMA"):
            assert ops.get(op, 0) == 0, (name, dt, op, ops.get(op))
        if dt == "f32" and name == "heat2d":      # temporal blocking evaluates point pairs
            assert ops.get("FADD2", 0) > 0, (name, ops)


def test_no_paired_fma_in_any_golden_random_kernel(golden_random):
    """No kernel of the golden random set (divisions, scalars, locals, min/max/abs/sqrt)
    compiles to FFMA2 in fp32: a paired FMA can only come from contraction."""
    from paper_1502_03504_b200.ir import deserialize
    meta, _ = golden_random
    n = 0
    for m in meta[::2]:
        kir = deserialize(m["ir"])
        if kir.rank < 2:
            continue
        ops = _sass_opcodes(kir, "f32")
        assert ops.get("FFMA2", 0) == 0, (m["trial"], m["source"])
        n += 1
    assert n >= 20
