"""Debug: run golden random trial N with a chosen dtype/shape/halo; report ok/mismatch."""
import json, sys, pathlib, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import lope_oracle as O
from paper_1502_03504_b200 import runtime as R
from paper_1502_03504_b200.ir import deserialize
G = pathlib.Path(__file__).resolve().parent.parent / "tests" / "golden"
meta = json.loads((G / "random.json").read_text())
t = int(sys.argv[1]); dt = sys.argv[2]; shape = tuple(int(x) for x in sys.argv[3].split(",")); h = int(sys.argv[4])
m = meta[t]
kir = deserialize(m["ir"])
npdt = np.float32 if dt == "float32" else np.float64
k = R.CompiledKernel(kir, dt)
f = O.hash_field(shape, 3, npdt)
a = R.HaloArray(shape, [h] * kir.rank, [h] * kir.rank, dt)
a.set_interior(f)
R.launch(k, [a], None, m["scalars"])
got = a.get_interior()
want = O.periodic_apply(f, kir, m["scalars"], npdt)
print(sys.argv[1:], os.environ.get("LOPE_FORCE_GENERIC"), "ok" if O.equal_bits(got, want) else O.first_mismatch(got, want), flush=True)
