"""Debug: run one IR body (store expression given on the command line) on a 2D field, tiled path."""
import sys, pathlib, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import lope_oracle as O
from paper_1502_03504_b200 import runtime as R
from paper_1502_03504_b200.ir import deserialize
dt = sys.argv[1]; expr = sys.argv[2]
text = f"LOPE1\nkernel k 2\narray u\nscalar c real\nscalar q integer\nstore u {expr}\nend\n"
kir = deserialize(text)
npdt = np.float32 if dt == "float32" else np.float64
k = R.CompiledKernel(kir, dt)
f = O.hash_field((40, 20), 3, npdt)
a = R.HaloArray((40, 20), [2, 2], [2, 2], dt)
a.set_interior(f)
sc = {"c": 0.75, "q": 3}
R.launch(k, [a], None, sc)
got = a.get_interior()
want = O.periodic_apply(f, kir, sc, npdt)
print(dt, repr(expr), "ok" if O.equal_bits(got, want) else O.first_mismatch(got, want), flush=True)
