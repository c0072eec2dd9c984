"""Child process of test_gpu_comm.py: P slab images through the C-ABI communicator in
one process (``dist.CommMultiSlab``), each case against the undecomposed run.

Run in its own process so ``CUDA_DEVICE_MAX_CONNECTIONS`` (one hardware queue per
image stream) is set before CUDA initialises; prints one JSON line per case.
"""

import json
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])

from oracle import lope_oracle as O  # noqa: E402
from paper_1502_03504_b200 import dist as D  # noqa: E402
from paper_1502_03504_b200 import runtime as R  # noqa: E402
from paper_1502_03504_b200 import stencils  # noqa: E402

CASES = [("lap3d7", (64, 48, 32), "float32", 2, 5), ("lap3d7", (64, 48, 32), "float32", 4, 4),
         ("heat2d", (128, 96), "float32", 3, 6), ("heat2d", (128, 96), "float64", 2, 1),
         ("box5x5", (64, 80), "float64", 4, 5), ("ninept2d", (96, 64), "float32", 8, 3),
         ("lap3d7", (32, 16, 24), "float64", 1, 3)]


def main():
    import torch
    for name, shape, dt, p, steps in CASES:
        kir = stencils.by_name(name)
        npdt = np.float32 if dt == "float32" else np.float64
        fp = kir.footprints[kir.array_params[0]].dims
        lo, hi = [a for a, _ in fp], [b for _, b in fp]
        k = R.CompiledKernel(kir, dt)
        field = O.hash_field(shape, 17, npdt)
        ms = D.CommMultiSlab(k, shape, lo, hi, dt, p)
        ms.set_global(field)
        ms.iterate(steps)
        torch.cuda.synchronize()
        got = ms.get_global()
        want = field
        for _ in range(steps):
            want = O.periodic_apply(want, kir, None, npdt)
        infos = [c.info() for c in ms.comms]
        ms.close()
        print(json.dumps({"case": [name, list(shape), dt, p, steps], "equal": O.equal_bits(got, want),
                          "epochs": [i["epoch"] for i in infos], "transport": infos[0]["transport"]}),
              flush=True)


if __name__ == "__main__":
    main()
