"""Throughput of the drop-in GPU Machine (paper_1502_03504_b200.machine.Machine) next to
the reference's own lopec.Machine on the same program and field: config 1's heat
program (1024^2, HALO_TRANSFER + launch per iteration, runtime.py:308-337) and config
2's 9-point program on 4096^2 (the 3-D programs have no driver loop), fp64 (the
reference's precision) and fp32, with 1 and 4 (2 x 2) images.  Wall time of Machine.run() (host field in; device twins built lazily), then
gather(); the GPU result is checked against the reference's bit for bit in fp64.
One JSON line per case.
    python tools/machine_bench.py [--steps 100] [--ref-steps 10]"""
import argparse
import json
import pathlib
import sys
import time

import numpy as np

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
for c in (REPO / "baseline" / "_ref",):
    if (c / "lopec" / "__init__.py").exists():
        sys.path.insert(0, str(c))

import lopec  # noqa: E402
from lopec.runtime import Machine as RefMachine, RunConfig  # noqa: E402

from oracle import lope_oracle as O  # noqa: E402  (input field only)
from oracle.lope_programs import program_text  # noqa: E402
from paper_1502_03504_b200.machine import Machine as GpuMachine  # noqa: E402


def check(kernel):
    prog, diags = lopec.parse_source(program_text(kernel), f"{kernel}.lope")
    if prog is None or diags:
        raise SystemExit(f"frontend rejected {kernel}: {diags}")
    return lopec.check_program(prog)


def timed_run(make):
    m = make()
    t0 = time.perf_counter()
    m.run()
    out = m.gather()
    return out, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--ref-steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    for kernel, shape in (("heat2d", (1024, 1024)), ("ninept2d", (4096, 4096))):
        chk = check(kernel)
        field = np.asfortranarray(O.hash_field(shape, 3, np.float64))
        pts = int(np.prod(shape))
        for images, rows in ((1, 1), (4, 2)):
            cfg = dict(images=images, grid_rows=rows)
            # reference: a few steps (it runs ~0.03-0.1 Gpts/s on one host thread)
            ref_out, ref_s = timed_run(lambda: RefMachine(chk, RunConfig(steps=a.ref_steps, **cfg), field.copy()))
            for dt in ("float64", "float32"):
                GpuMachine(chk, RunConfig(steps=2, **cfg), field.copy(), dtype=dt).run()     # compile, warm
                torch.cuda.synchronize()
                out, el = timed_run(lambda: GpuMachine(chk, RunConfig(steps=a.steps, **cfg), field.copy(),
                                                        dtype=dt))
                # marginal cost of a step: the same run with 5x the steps (the one-time host
                # scatter of the input field in lopec's own _alloc_host, uploads and the final
                # gather cancel out)
                _, el5 = timed_run(lambda: GpuMachine(chk, RunConfig(steps=5 * a.steps, **cfg), field.copy(),
                                                       dtype=dt))
                step_ms = 1e3 * (el5 - el) / (4 * a.steps)
                chk_bits = None
                if dt == "float64":
                    g_out, _ = timed_run(lambda: GpuMachine(chk, RunConfig(steps=a.ref_steps, **cfg), field.copy(),
                                                             dtype=dt))
                    chk_bits = bool(O.equal_bits(np.asarray(g_out), np.asarray(ref_out)))
                print(json.dumps({
                    "program": kernel, "shape": list(shape), "images": images, "grid_rows": cfg["grid_rows"],
                    "dtype": dt, "steps": a.steps, "gpu_machine_s": round(el, 4),
                    "gpu_machine_gpts": round(pts * a.steps / el / 1e9, 3),
                    "gpu_machine_marginal_ms_per_step": round(step_ms, 4),
                    "gpu_machine_marginal_gpts": round(pts / (step_ms * 1e-3) / 1e9, 2) if step_ms > 0 else None,
                    "reference_machine_steps": a.ref_steps, "reference_machine_s": round(ref_s, 3),
                    "reference_machine_gpts": round(pts * a.ref_steps / ref_s / 1e9, 4),
                    "bitwise_equal_to_reference_fp64": chk_bits,
                    "timed": "Machine(...).run() + gather(), host field in and out (wall clock)"}), flush=True)


if __name__ == "__main__":
    main()
