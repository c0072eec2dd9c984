"""The drop-in Machine (paper_1502_03504_b200.machine) against the reference Machine.

For programs run on the reference Machine when the fixtures were made
(tests/golden/machine.*: several kernels, image grids, device subimages), the GPU
Machine must reproduce the gathered field, every image's padded block, the
per-image counters and the event log exactly.
"""

import numpy as np
import pytest

from conftest import import_lopec, load_json, load_npz

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)
if not import_lopec():
    pytest.skip("the reference package lopec is not importable (baseline/_ref)", allow_module_level=True)

from lopec import check_program, parse_source  # noqa: E402
from lopec.runtime import RunConfig  # noqa: E402

from oracle import lope_oracle as O  # noqa: E402
from paper_1502_03504_b200.machine import Machine  # noqa: E402

CASES = load_json("machine.json")
ARR = load_npz("machine.npz")


def compile_text(text):
    program, diags = parse_source(text, "test.lope")
    assert program is not None and not diags
    result = check_program(program)
    assert result.ok
    return result


def _device_maps():
    """One GPU per image (as many as the node has), and the mapping forced onto the
    first GPU twice (images alternate between two 'devices': the cross-device code
    path -- per-device launches, events between streams, destination-side copies --
    runs even on a one-GPU box)."""
    n = torch.cuda.device_count()
    maps = [None, [0, 0]]
    if n > 1:
        maps.append(list(range(n)))
    return maps


@pytest.mark.parametrize("devices", _device_maps(), ids=lambda d: "auto" if d is None else "dev" + "".join(map(str, d)))
@pytest.mark.parametrize("case", CASES, ids=[c["tag"] for c in CASES])
def test_gpu_machine_reproduces_reference_machine(case, devices):
    result = compile_text(case["text"])
    field = ARR[case["tag"] + "_in"]
    m = Machine(result, RunConfig(images=case["images"], grid_rows=case["grid_rows"],
                                  devices=case["devices"], steps=case["steps"]), field.copy(), devices=devices)
    if devices is not None:
        assert [m.device_of(k) for k in m.images] == [devices[(k - 1) % len(devices)] for k in m.images]
    m.run()
    assert np.array_equal(m.gather(), ARR[case["tag"] + "_out"])
    for k in m.images:
        assert np.array_equal(m.arrays["u"].view(k), ARR[f"{case['tag']}_blk{k}"]), k
    assert {str(k): v for k, v in m.counters.items()} == case["counters"]
    assert [list(e) for e in m.events] == case["events"]


def test_gpu_machine_orders_are_bitwise_identical():
    case = next(c for c in CASES if c["kernel"] == "skew")
    result = compile_text(case["text"])
    field = ARR[case["tag"] + "_in"]
    outs = []
    for order, seed in (("vector", None), ("forward", None), ("reverse", None), ("shuffle", 3)):
        m = Machine(result, RunConfig(images=2, grid_rows=2, steps=3, order=order, shuffle_seed=seed),
                    field.copy())
        m.run()
        outs.append(m.gather())
    assert all(np.array_equal(o, outs[0]) for o in outs)


def test_gpu_machine_fp32_matches_restatement():
    case = next(c for c in CASES if c["kernel"] == "fig1" and c["images"] == 1)
    result = compile_text(case["text"])
    field = ARR[case["tag"] + "_in"]
    m = Machine(result, RunConfig(images=2, grid_rows=2, steps=3), field.copy(), dtype="float32")
    m.run()
    from paper_1502_03504_b200.ir import from_lopec
    from lopec.ir import lower_kernel
    kir = from_lopec(lower_kernel(result.kernels["fig1"]))
    want = field.astype(np.float32)
    for _ in range(3):
        want = O.periodic_apply(want, kir, None, np.float32)
    assert O.equal_bits(m.gather().astype(np.float32), want)


def test_cli_run_matches_reference_output(tmp_path, capsys):
    """``python -m paper_1502_03504_b200.cli run`` prints exactly what ``lopec run``
    prints for the same program (the reference Machine's gathered field, %.17g)."""
    import io
    from lopec.arrayio import write_array
    from paper_1502_03504_b200 import cli
    for case in CASES:
        src = tmp_path / f"{case['tag']}.lope"
        src.write_text(case["text"])
        fin = tmp_path / f"{case['tag']}.in"
        buf = io.StringIO()
        write_array(buf, ARR[case["tag"] + "_in"])
        fin.write_text(buf.getvalue())
        out = tmp_path / f"{case['tag']}.out"
        rc = cli.main(["run", str(src), "--images", str(case["images"]), "--grid-rows",
                       str(case["grid_rows"]), "--devices", str(case["devices"]), "--steps", str(case["steps"]),
                       "--input", str(fin),
                       "-o", str(out)])
        assert rc == 0
        want = io.StringIO()
        write_array(want, ARR[case["tag"] + "_out"])
        assert out.read_text() == want.getvalue(), case["tag"]
