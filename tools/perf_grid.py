"""MP x NP (and P0 x P1 x P2) image grids on one GPU: every image's
block of a CartGrid in HBM, faces moved between blocks with lope_copy_box in the
reference's exchange order (dist.MultiGrid), against the same domain as one block.
A one-GPU proxy for the grid pipeline's overhead (extra launches, strided face copies,
smaller blocks), not a multi-GPU measurement; every result is also checked bit for bit
against the undecomposed run.  One JSON line per case.
    python tools/perf_grid.py [--steps 20]"""
import argparse
import json
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import lope_oracle as O  # noqa: E402  (input field only)
from paper_1502_03504_b200 import dist as D  # noqa: E402
from paper_1502_03504_b200 import runtime as R  # noqa: E402
from paper_1502_03504_b200 import stencils  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    cases = [("ninept2d", (8192, 8192), "float32", [(2, 2), (4, 2), (1, 4)]),
             ("box5x5", (8192, 8192), "float64", [(2, 2), (1, 8)]),
             ("lap3d7", (512, 512, 512), "float32", [(2, 2, 2), (1, 2, 4)])]
    for name, shape, dt, splits_list in cases:
        kir = stencils.by_name(name)
        k = R.CompiledKernel(kir, dt)
        fp = kir.footprints[kir.array_params[0]].dims
        lo, hi = [n for n, _ in fp], [p for _, p in fp]
        npdt = np.float32 if dt == "float32" else np.float64
        field = O.hash_field(shape, 9, npdt)
        base = R.HaloArray(shape, lo, hi, dt)
        base.set_interior(field)
        R.iterate(k, base, 2)                                   # compile / plans
        base.set_interior(field)
        ms_single = timed(lambda: R.iterate(k, base, a.steps))
        want = base.get_interior()
        pts = int(np.prod(shape)) * a.steps
        for splits in splits_list:
            mg = D.MultiGrid(k, D.CartGrid(shape, list(splits), lo, hi), dt)
            mg.set_global(field)
            mg.iterate(2)
            mg.set_global(field)
            ms = timed(lambda: mg.iterate(a.steps))
            got = mg.get_global()
            print(json.dumps({"kernel": name, "shape": list(shape), "dtype": dt, "splits": list(splits),
                              "steps": a.steps, "ms_grid": round(ms, 3), "gpts_grid": round(pts / ms / 1e6, 1),
                              "ms_single_block": round(ms_single, 3),
                              "gpts_single_block": round(pts / ms_single / 1e6, 1),
                              "bitwise_equal": bool(O.equal_bits(got, want))}), flush=True)
            del mg
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
