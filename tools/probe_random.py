"""Debug: run each golden random kernel one by one (CUDA_LAUNCH_BLOCKING=1) and report."""
import json, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import lope_oracle as O
from paper_1502_03504_b200 import runtime as R
from paper_1502_03504_b200.ir import deserialize
G = pathlib.Path(__file__).resolve().parent.parent / "tests" / "golden"
meta = json.loads((G / "random.json").read_text())
arrs = np.load(G / "random.npz")
only = int(sys.argv[1]) if len(sys.argv) > 1 else None
for m in meta:
    if only is not None and m["trial"] != only:
        continue
    kir = deserialize(m["ir"])
    dts = (("float64", np.float64), ("float32", np.float32))
    if len(sys.argv) > 2:
        dts = [d for d in dts if d[0] == sys.argv[2]]
    for dt, npdt in dts:
        k = R.CompiledKernel(kir, dt)
        print("trial", m["trial"], dt, "rank", kir.rank, k.describe(), flush=True)
        f = arrs[f"r{m['trial']}_in"].astype(npdt)
        a = R.HaloArray(f.shape, [2] * kir.rank, [2] * kir.rank, dt)
        a.set_interior(f)
        R.iterate(k, a, 1, m["scalars"])
        got = a.get_interior()
        want = arrs[f"r{m['trial']}_out"] if dt == "float64" else O.periodic_apply(f, kir, m["scalars"], npdt)
        print("   ok" if O.equal_bits(got, want) else f"   MISMATCH {O.first_mismatch(got, want)}", flush=True)
