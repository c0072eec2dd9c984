"""Throughput of the shapes that used to drop to the generic kernel:
ragged x (lap3d7 1001^3 fp32), a two-array kernel at 1024^3 (fused steps on the
multi-array TMA kernel), rank 1 (avg3, 2^28 cells fp64).  One JSON line per case:
fused steps timed with CUDA events after warm-up, algorithmic bytes = (arrays read +
arrays stored) x sizeof(T) x points, against MEASURED_PEAKS.json hbm_gbs.
    python tools/perf_cliffs.py [--steps 20]"""
import argparse
import json
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import torch  # noqa: E402

from paper_1502_03504_b200 import runtime as R, stencils  # noqa: E402
from paper_1502_03504_b200.ir import KernelBuilder  # noqa: E402


def peak():
    try:
        return float(json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 7672.0


def two_array_3d():
    kb = KernelBuilder("two3d", 3)
    u, v = kb.array("u"), kb.array("v")
    kb.store(u, u[0, 0, 0] + 0.125 * (u[-1, 0, 0] + u[1, 0, 0] + u[0, -1, 0] + u[0, 1, 0]
                                      + u[0, 0, -1] + u[0, 0, 1] - 6 * u[0, 0, 0]) + 0.5 * v[0, 0, 0])
    return kb.build()


def timed(fn, steps, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record()
    for i in range(steps):
        fn()
        evs[i + 1].record()
    torch.cuda.synchronize()
    ms = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(steps))
    return ms[len(ms) // 2], ms[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cases", default="ragged3d,aligned3d,two3d,rank1")
    a = ap.parse_args()
    pk = peak()
    cases = a.cases.split(",")
    for case in cases:
        torch.cuda.empty_cache()
        if case in ("ragged3d", "aligned3d"):
            shape = (1001, 1001, 1001) if case == "ragged3d" else (1024, 1024, 1024)
            kir, dt, narr = stencils.lap3d7(), "float32", (1, 1)
            k = R.CompiledKernel(kir, dt)
            arr = R.HaloArray(shape, (1, 1, 1), (1, 1, 1), dt)
            arr.fill_hash(1)
            arr.spare()
            R.halo_transfer(arr)
            k.tune(arr)                       # the plan tuner's pick for this geometry
            fn = lambda: R.step(k, arr)  # noqa: E731
        elif case == "two3d":
            shape = (1024, 1024, 1024)
            kir, dt, narr = two_array_3d(), "float32", (2, 1)
            k = R.CompiledKernel(kir, dt)
            hs = [R.HaloArray(shape, (1, 1, 1), (1, 1, 1), dt) for _ in range(2)]
            for h in hs:
                h.data.uniform_(-1, 1)
                R.halo_transfer(h)
            hs[0].spare()
            fn = lambda: R.step_arrays(k, hs)  # noqa: E731
        elif case == "rank1":
            shape = (1 << 28,)
            kir, dt, narr = stencils.avg3(), "float64", (1, 1)
            k = R.CompiledKernel(kir, dt)
            arr = R.HaloArray(shape, (1,), (1,), dt)
            arr.data.uniform_(-1, 1)
            arr.spare()
            R.halo_transfer(arr)
            fn = lambda: R.step(k, arr)  # noqa: E731
        else:
            raise SystemExit(f"unknown case {case}")
        ms, ms_min = timed(fn, a.steps)
        pts = 1
        for s in shape:
            pts *= s
        esz = 4 if dt == "float32" else 8
        alg = (narr[0] + narr[1]) * esz * pts
        gbs = alg / (ms * 1e-3) / 1e9
        print(json.dumps({"case": case, "kernel": kir.name, "shape": list(shape), "dtype": dt,
                          "ms_median": round(ms, 4), "ms_min": round(ms_min, 4),
                          "alg_bytes": alg, "alg_gbs": round(gbs, 1), "frac_of_peak": round(gbs / pk, 4),
                          "peak_gbs": pk, "launches": json.loads(k.describe())["launches"]}), flush=True)


if __name__ == "__main__":
    main()
