"""Constant-divisor division (LopeAr::divc) is bit-identical to IEEE division.

The code generator turns ``x / c`` for a non-power-of-two constant ``c`` into a
reciprocal multiply plus an FMA correction (Markstein), with IEEE division kept for
0, inf, NaN and the extreme exponent ranges.  These tests run ``u / c`` through the
product path (lope_launch) on inputs that cover every exponent, the special values
and, for fp32, every significand of a binade, and compare the bits with numpy's
correctly rounded division (the reference's arithmetic, lopec/ir.py:290).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle.lope_oracle import equal_bits

pytestmark = pytest.mark.gpu

DIVISORS = [25.0, 3.0, 7.0, 10.0, 0.1, 1.0 / 3.0, -9.5, 12345.678, 1e-5, 3e7, 1e300]


def _kernel(c):
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder("divc", 2)
    u = kb.array("u")
    kb.store(u, u[0, 0] / c)
    return kb.build()


def _random_bits(rng, n, dtype):
    if dtype == np.float64:
        bits = rng.integers(0, 2**63, size=n, dtype=np.uint64) | (rng.integers(0, 2, size=n, dtype=np.uint64) << 63)
        x = bits.view(np.float64)
    else:
        bits = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        x = bits.view(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0], dtype=dtype)
    fi = np.finfo(dtype)
    special = np.concatenate([special, np.array([fi.tiny, -fi.tiny, fi.max, -fi.max, fi.smallest_subnormal,
                                                 fi.tiny * 3, fi.eps], dtype=dtype)])
    x[:special.size] = special
    return x


def _run(c, x2d, dtype_name):
    from paper_1502_03504_b200 import runtime as R
    k = R.CompiledKernel(_kernel(c), dtype_name)
    arr = R.HaloArray(x2d.shape, [0, 0], [0, 0], dtype_name)
    arr.set_interior(x2d)
    R.launch(k, [arr])
    return arr.get_interior()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_divc_random_bits_all_exponents(dtype):
    rng = np.random.default_rng(7)
    shape = (2048, 1024)
    x = _random_bits(rng, shape[0] * shape[1], dtype).reshape(shape, order="F")
    name = "float64" if dtype == np.float64 else "float32"
    for c in DIVISORS:
        with np.errstate(all="ignore"):
            want = (x / dtype(c)).astype(dtype)
        got = _run(c, x, name)
        assert equal_bits(got, want), f"{name} x/{c!r}: first mismatch at {np.argwhere(~((got == want) | (np.isnan(got) & np.isnan(want))))[:3]}"


def test_divc_fp32_every_significand():
    # all 2^23 significands of [1, 2) and of a binade near the fast path's lower bound
    m = np.arange(1 << 23, dtype=np.uint32)
    for exp_bits in (127, 127 - 89, 127 + 89):
        x = ((np.uint32(exp_bits) << np.uint32(23)) | m).view(np.float32).reshape((8192, 1024), order="F")
        for c in (25.0, 3.0, 10.0, 0.1, -9.5):
            want = (x / np.float32(c)).astype(np.float32)
            assert equal_bits(_run(c, x, "float32"), want), f"binade {exp_bits}, c={c}"


def test_divc_fp64_near_halfway_quotients():
    # x = c * q + tiny: quotients just off the representable grid, the hard cases
    rng = np.random.default_rng(11)
    n = 1 << 21
    for c in (25.0, 3.0, 7.0, 10.0):
        q = rng.uniform(1.0, 2.0, size=n)
        x = q * c
        x = np.nextafter(x, np.where(rng.integers(0, 2, size=n) == 1, np.inf, -np.inf))
        x = x.reshape((2048, 1024), order="F")
        want = x / c
        assert equal_bits(_run(c, x, "float64"), want), f"c={c}"


def _wide_range_field(rng, shape, dtype):
    """U(-1,1) scaled by 2^e with e spread over the whole exponent range, plus zeros,
    infinities and subnormals -- so sums land in the fast, tiny and huge ranges."""
    fi = np.finfo(dtype)
    lo_e, hi_e = (-1070, 1020) if dtype == np.float64 else (-145, 125)
    # magnitude set per plane (whole stencils go tiny / huge) with a little jitter
    plane_e = np.round(np.linspace(lo_e, hi_e, shape[-1])).astype(np.int64)
    e = plane_e.reshape((1,) * (len(shape) - 1) + (-1,)) + rng.integers(-3, 4, size=shape)
    x = (rng.uniform(-1, 1, size=shape) * np.exp2(e.astype(np.float64))).astype(dtype)
    flat = x.reshape(-1, order="F")
    idx = rng.choice(flat.size, size=16, replace=False)
    flat[idx[:4]] = 0.0
    flat[idx[4:6]] = np.inf
    flat[idx[6:8]] = -np.inf
    flat[idx[8:12]] = fi.smallest_subnormal
    return flat.reshape(shape, order="F")


@pytest.mark.parametrize("force_generic", [False, True])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_divc_in_zstar_stencil_matches_oracle(monkeypatch, dtype, force_generic):
    """3-D z-star stencil / 7 (tiled path keeps past planes in registers) with operands
    in every range: the fast points and the re-evaluated slow points both match the
    restatement bit for bit, on the tiled and on the generic kernel."""
    from oracle import lope_oracle as O
    from paper_1502_03504_b200 import runtime as R
    from paper_1502_03504_b200.ir import KernelBuilder
    if force_generic:
        monkeypatch.setenv("LOPE_FORCE_GENERIC", "1")
    kb = KernelBuilder("lap7div", 3)
    u = kb.array("u")
    s = u[-1, 0, 0] + u[1, 0, 0] + u[0, -1, 0] + u[0, 1, 0] + u[0, 0, -1] + u[0, 0, 1] + u[0, 0, 0]
    kb.store(u, s / 7.0)
    kir = kb.build()
    npd = np.float64 if dtype == "float64" else np.float32
    rng = np.random.default_rng(5)
    field = _wide_range_field(rng, (64, 24, 20), npd)
    k = R.CompiledKernel(kir, dtype)
    arr = R.HaloArray(field.shape, [1, 1, 1], [1, 1, 1], dtype)
    arr.set_interior(field)
    R.halo_transfer(arr)
    R.step(k, arr)
    with np.errstate(all="ignore"):
        want = O.periodic_apply(field, kir, dtype=npd)
    assert O.equal_bits(arr.get_interior(), want), O.first_mismatch(arr.get_interior(), want)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_box5x5_wide_range_matches_oracle(dtype):
    """Config 4's kernel ((sum of 25)/25) on operands spanning every range."""
    from oracle import lope_oracle as O
    from paper_1502_03504_b200 import runtime as R, stencils
    kir = stencils.box5x5()
    npd = np.float64 if dtype == "float64" else np.float32
    field = _wide_range_field(np.random.default_rng(9), (256, 96), npd)
    arr = R.HaloArray(field.shape, [2, 2], [2, 2], dtype)
    arr.set_interior(field)
    R.halo_transfer(arr)
    R.step(R.CompiledKernel(kir, dtype), arr)
    with np.errstate(all="ignore"):
        want = O.periodic_apply(field, kir, dtype=npd)
    assert O.equal_bits(arr.get_interior(), want), O.first_mismatch(arr.get_interior(), want)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_scalar_divisor_matches_ieee(dtype):
    """x / s for a kernel scalar s (host-side reciprocal, NaN for unsafe s)."""
    from paper_1502_03504_b200 import runtime as R
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder("divs", 2)
    u = kb.array("u")
    s = kb.scalar("s")
    kb.store(u, (u[0, 0] + u[1, 0]) / s)
    kir = kb.build()
    name = "float64" if dtype == np.float64 else "float32"
    k = R.CompiledKernel(kir, name)
    rng = np.random.default_rng(3)
    shape = (1024, 512)
    x = _random_bits(rng, shape[0] * shape[1], dtype).reshape(shape, order="F")
    for sv in (25.0, 0.1, -3.0, 7.0, 0.0, 1e-30, 3e20, float("inf"), float("nan")):
        arr = R.HaloArray(shape, [0, 0], [1, 0], name)
        arr.set_interior(x)
        R.halo_transfer(arr)
        R.launch(k, [arr], scalars={"s": sv})
        with np.errstate(all="ignore"):
            xr = np.roll(x, -1, axis=0)
            want = ((x + xr) / dtype(sv)).astype(dtype)
        got = arr.get_interior()
        assert equal_bits(got, want), f"s={sv}: {np.argwhere(~((got == want) | (np.isnan(got) & np.isnan(want))))[:3]}"
