"""Slab-decomposed pipeline on one GPU: P in-process slabs (boundary planes, face
spans, ring exchange) must give bit-identical fields to the undecomposed run, the
reference's decomposition invariance (tests/test_runtime.py:90-98 there)."""

import numpy as np
import pytest

from oracle import lope_oracle as O
from paper_1502_03504_b200 import stencils

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1502_03504_b200 import dist as D  # noqa: E402
from paper_1502_03504_b200 import runtime as R  # noqa: E402


def halos(kir):
    fp = kir.footprints[kir.array_params[0]].dims
    return [n for n, _ in fp], [p for _, p in fp]


@pytest.mark.parametrize("name,shape,dt,ps", [
    ("lap3d7", (64, 40, 48), "float32", (2, 3, 4, 8)),
    ("box5x5", (96, 64), "float64", (2, 4, 8)),
    ("drift2", (64, 48), "float32", (2, 4)),
    ("heat2d", (256, 128), "float64", (2, 4, 8)),
])
def test_slab_decomposition_is_bitwise_invariant(name, shape, dt, ps):
    kir = stencils.by_name(name)
    lo, hi = halos(kir)
    npdt = np.float32 if dt == "float32" else np.float64
    sc = {"c": 0.25} if name == "drift2" else None
    field = O.hash_field(shape, 31, npdt)
    k = R.CompiledKernel(kir, dt)
    base = R.HaloArray(shape, lo, hi, dt)
    base.set_interior(field)
    R.iterate(k, base, 5, sc)
    want = base.get_interior()
    ref = field
    for _ in range(5):
        ref = O.periodic_apply(ref, kir, sc, npdt)
    assert O.equal_bits(want, ref)
    for p in ps:
        ms = D.MultiSlab(k, shape, lo, hi, dt, p, sc)
        ms.set_global(field)
        ms.iterate(5)
        got = ms.get_global()
        assert O.equal_bits(got, want), (name, p, O.first_mismatch(got, want))


def test_single_rank_stepper_matches_runtime():
    kir = stencils.lap3d7()
    shape = (128, 64, 32)
    field = O.hash_field(shape, 3, np.float32)
    k = R.CompiledKernel(kir, "float32")
    arr = D.SlabArray(shape, (1, 1, 1), (1, 1, 1), "float32")
    arr.block.set_interior(field)
    D.SlabStepper(k, arr).iterate(4)
    ref = field
    for _ in range(4):
        ref = O.periodic_apply(ref, kir, None, np.float32)
    assert O.equal_bits(arr.block.get_interior(), ref)
