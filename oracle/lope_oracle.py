"""CPU oracle for the LOPe stencil hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` / ``--impl reference``) may import this module, and only as
the checker or the timed CPU reference.  The product path
(``paper_1502_03504_b200``) never calls it and fails loudly without its CUDA
library.

It restates, in numpy, the reference algorithm of ``/root/reference/pkg``:

* ``run_body``        — ``lopec/ir.py:258-308`` (tree walk; per-node numpy op),
                        parameterised by dtype.  With ``np.float64`` it is the
                        reference's own arithmetic; with ``np.float32`` it is the
                        fp32 restatement SURVEY §8(c) requires (F3: the reference
                        computes only fp64).  Constants are ``dtype(value)``,
                        scalars are cast to ``dtype`` (integer scalars included).
* ``periodic_apply``  — ``lopec/runtime.py:744-765`` (``oracle_step``: dense
                        ``np.roll`` reads, rank-agnostic).
* ``periodic_apply_planes`` — the same result restricted to a slab of the
                        slowest axis, reading only the planes it needs (exact
                        for full-size sampled checks).
* ``halo_fill``       — ``lopec/runtime.py:643-697`` with every neighbour equal to
                        self (P = 1): per dim ascending, low halo <- high
                        interior, high halo <- low interior, full padded slabs.
* ``launch``          — ``lopec/runtime.py:541-618``: snapshot reads, pending
                        centre values stored over the (1-based, inclusive)
                        launch range; everything else unchanged.
* ``machine_run``     — one image running ``do it=1,nsteps; HALO_TRANSFER;
                        do concurrent ... end do`` (``corpus/*.lope``).
* ``exchange_blocks`` — ``runtime.py:643-697`` over a 1-D ring of images along the
                        slowest axis (slab decomposition).
* ``hash_field``      — the decomposition-independent synthetic input
                        (splitmix64 of the global linear index).

Parity is pinned by ``tests/golden/*.npz`` (generated from the reference itself
by ``tests/golden/gen_golden.py``) — see ``tests/test_oracle.py``.
"""

from __future__ import annotations

import functools
import math

import numpy as np

_ADD, _MUL, _DIV, _NEG = "Add", "Mul", "Div", "Neg"


def run_body(kir, read, scalars=None, dtype=np.float64):
    """Evaluate ``kir.body``; returns ``{array: pending centre values}`` (ir.py:258-308)."""
    dt = np.dtype(dtype).type
    env = {k: dt(v) for k, v in (scalars or {}).items()}
    pending = {}

    def ev(e):
        cls = type(e).__name__
        if cls == "Const":
            return dt(e.value)
        if cls == "ScalarRead":
            if e.name not in env:
                raise KeyError(f"kernel local '{e.name}' read before assignment")
            return env[e.name]
        if cls == "Read":
            if e.array in pending and all(o == 0 for o in e.offsets):
                return pending[e.array]
            return read(e.array, tuple(e.offsets))
        if cls == _ADD:
            return ev(e.left) + ev(e.right)
        if cls == _MUL:
            return ev(e.left) * ev(e.right)
        if cls == _DIV:
            return ev(e.left) / ev(e.right)
        if cls == _NEG:
            return -ev(e.operand)
        if cls == "IntrinsicCall":
            args = [ev(a) for a in e.args]
            if e.fn == "abs":
                return np.abs(args[0])
            if e.fn == "sqrt":
                return np.sqrt(args[0])
            if e.fn == "min":
                return functools.reduce(np.minimum, args)
            if e.fn == "max":
                return functools.reduce(np.maximum, args)
        raise TypeError(f"cannot evaluate {cls}")

    with np.errstate(all="ignore"):
        for st in kir.body:
            v = ev(st.expr)
            if st.is_array:
                pending[st.target] = v
            else:
                env[st.target] = v
    return pending


def periodic_apply(field, kir, scalars=None, dtype=np.float64):
    """One dense periodic application of ``kir`` (oracle_step, runtime.py:744-765)."""
    work = np.asarray(field).astype(dtype, copy=True)
    axes = tuple(range(work.ndim))

    def read(name, offsets):
        if all(o == 0 for o in offsets):
            return work.copy()
        return np.roll(work, shift=tuple(-o for o in offsets), axis=axes)

    pending = run_body(kir, read, scalars, dtype)
    return np.asarray(pending[kir.stored_arrays[0]], dtype=dtype)


def periodic_apply_planes(get_planes, shape, kir, z0, z1, scalars=None, dtype=np.float64):
    """Rows/planes ``z0:z1`` (last axis) of ``periodic_apply`` without the whole field.

    ``get_planes(idx)`` returns the field restricted to last-axis indices ``idx``
    (a 1-D int array, already wrapped modulo the extent).
    """
    fp = kir.footprints[kir.array_params[0]].dims
    zn, zp = fp[-1]
    n = shape[-1]
    idx = np.arange(z0 - zn, z1 + zp) % n
    slab = np.asarray(get_planes(idx)).astype(dtype, copy=False)
    inner = tuple(range(slab.ndim - 1))

    def read(name, offsets):
        *oin, oz = offsets
        s = slab[..., zn + oz: zn + oz + (z1 - z0)]
        if any(o != 0 for o in oin):
            s = np.roll(s, shift=tuple(-o for o in oin), axis=inner)
        return s.copy()

    pending = run_body(kir, read, scalars, dtype)
    return np.asarray(pending[kir.stored_arrays[0]], dtype=dtype)


def periodic_apply_planes_steps(get_planes, shape, kir, z0, z1, steps, scalars=None, dtype=np.float64):
    """Planes ``z0:z1`` (last axis) after ``steps`` applications of ``periodic_apply``.

    Reads the window of planes the result depends on (``steps`` footprints beyond
    each end, wrapped modulo the extent) and applies the kernel ``steps`` times, the
    window shrinking by one footprint per step; the inner axes are whole and
    periodic.  ``steps = 1`` is ``periodic_apply_planes``.  Sizes up to the full
    BASELINE configurations stay a few planes of host memory.
    """
    fp = kir.footprints[kir.array_params[0]].dims
    zn, zp = fp[-1]
    n = shape[-1]
    if steps <= 0:
        return np.asarray(get_planes(np.arange(z0, z1) % n)).astype(dtype, copy=False)
    slab = np.asarray(get_planes(np.arange(z0 - steps * zn, z1 + steps * zp) % n)).astype(dtype, copy=True)
    inner = tuple(range(slab.ndim - 1))
    for _ in range(steps):
        nout = slab.shape[-1] - zn - zp
        cur = slab

        def read(name, offsets, cur=cur, nout=nout):
            *oin, oz = offsets
            s = cur[..., zn + oz: zn + oz + nout]
            if any(o != 0 for o in oin):
                s = np.roll(s, shift=tuple(-o for o in oin), axis=inner)
            return s.copy()

        slab = np.asarray(run_body(kir, read, scalars, dtype)[kir.stored_arrays[0]], dtype=dtype)
    return slab


def padded_shape(interior, lo, hi):
    return tuple(m + a + b for m, a, b in zip(interior, lo, hi))


def embed(field, lo, hi, dtype=None):
    """Place a global interior into a zero padded block (_alloc_host + _scatter_block)."""
    field = np.asarray(field)
    dtype = dtype or field.dtype
    out = np.zeros(padded_shape(field.shape, lo, hi), dtype=dtype)
    out[tuple(slice(a, a + m) for a, m in zip(lo, field.shape))] = field
    return out


def interior(padded, lo, hi):
    return padded[tuple(slice(a, s - b) for a, b, s in zip(lo, hi, padded.shape))]


def halo_fill(padded, lo, hi, dims=None):
    """Periodic halo exchange of one image with itself, in place (runtime.py:653-697)."""
    rank = padded.ndim
    for d in range(rank):
        if dims is not None and d not in dims:
            continue
        wl, wh = lo[d], hi[d]
        if wl == 0 and wh == 0:
            continue
        m = padded.shape[d] - wl - wh

        def slab(a, b):
            idx = [slice(None)] * rank
            idx[d] = slice(a, b)
            return tuple(idx)

        low_halo, high_halo = slab(0, wl), slab(wl + m, wl + m + wh)
        low_int, high_int = slab(wl, wl + wh), slab(m, m + wl)
        if wl:
            padded[low_halo] = padded[high_int].copy()
        if wh:
            padded[high_halo] = padded[low_int].copy()
    return padded


def launch(buffers, lo_hi, kir, ranges, scalars=None, dtype=np.float64):
    """``_launch`` + ``_launch_vector`` on padded blocks (runtime.py:594-618).

    ``buffers``: ``{array: padded ndarray}`` (modified in place, like the live
    buffers); ``lo_hi``: ``{array: (lo, hi)}``; ``ranges``: 1-based inclusive.
    """
    if any(a > b for a, b in ranges):
        return buffers
    snaps = {p: b.copy() for p, b in buffers.items()}

    def read(name, offsets):
        lo = lo_hi[name][0]
        return snaps[name][tuple(slice(a - 1 + h + o, b + h + o)
                                 for (a, b), h, o in zip(ranges, lo, offsets))]

    pending = run_body(kir, read, scalars, dtype)
    for name, v in pending.items():
        lo = lo_hi[name][0]
        buffers[name][tuple(slice(a - 1 + h, b + h) for (a, b), h in zip(ranges, lo))] = v
    return buffers


def machine_run(field, kir, steps, scalars=None, dtype=np.float64, lo=None, hi=None):
    """Single-image ``do it=1,nsteps; HALO_TRANSFER; launch(full interior)``; returns the padded block."""
    field = np.asarray(field).astype(dtype)
    fp = kir.footprints[kir.array_params[0]].dims
    lo = tuple(lo) if lo is not None else tuple(n for n, _ in fp)
    hi = tuple(hi) if hi is not None else tuple(p for _, p in fp)
    name = kir.array_params[0]
    blk = embed(field, lo, hi, dtype)
    ranges = [(1, m) for m in field.shape]
    for _ in range(steps):
        halo_fill(blk, lo, hi)
        launch({name: blk}, {name: (lo, hi)}, kir, ranges, scalars, dtype)
    return blk


def exchange_blocks(blocks, lo, hi, axis=-1):
    """Ring exchange of padded blocks decomposed along ``axis`` (runtime.py:653-697, MP=P).

    Non-decomposed dims are filled locally; the decomposed dim's halos come from
    the ring neighbours, sweeping dims in ascending order so corners follow.
    """
    p = len(blocks)
    rank = blocks[0].ndim
    axis = axis % rank
    for d in range(rank):
        wl, wh = lo[d], hi[d]
        if wl == 0 and wh == 0:
            continue
        if d != axis:
            for b in blocks:
                halo_fill(b, lo, hi, dims=(d,))
            continue
        m = blocks[0].shape[d] - wl - wh

        def slab(a, b):
            idx = [slice(None)] * rank
            idx[d] = slice(a, b)
            return tuple(idx)

        new = []
        for k in range(p):
            lowsrc = blocks[(k - 1) % p][slab(m, m + wl)].copy()
            highsrc = blocks[(k + 1) % p][slab(wl, wl + wh)].copy()
            new.append((lowsrc, highsrc))
        for k in range(p):
            if wl:
                blocks[k][slab(0, wl)] = new[k][0]
            if wh:
                blocks[k][slab(wl + m, wl + m + wh)] = new[k][1]
    return blocks


# ---------------------------------------------------------------------------
# Synthetic inputs

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def hash_values(linear_index, seed, dtype=np.float64):
    """U(-1,1) value of global column-major linear index ``i`` under ``seed``."""
    with np.errstate(over="ignore"):
        x = np.asarray(linear_index, dtype=np.uint64) + np.uint64(seed) * _GOLDEN
    z = splitmix64(x)
    v = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return (2.0 * v - 1.0).astype(dtype)


def hash_field(shape, seed, dtype=np.float64):
    """The whole synthetic field of ``shape`` (column-major global linear index)."""
    idx = np.zeros(shape, dtype=np.uint64)
    stride = 1
    for d, m in enumerate(shape):
        ar = np.arange(m, dtype=np.uint64) * np.uint64(stride)
        sh = [1] * len(shape)
        sh[d] = m
        idx = idx + ar.reshape(sh)
        stride *= m
    return hash_values(idx, seed, dtype)


def hash_planes(global_shape, seed, zidx, dtype=np.float64):
    """Planes ``zidx`` (last axis) of ``hash_field(global_shape, seed)`` without building it."""
    inner = global_shape[:-1]
    idx = np.zeros(tuple(inner) + (len(zidx),), dtype=np.uint64)
    stride = 1
    for d, m in enumerate(inner):
        ar = np.arange(m, dtype=np.uint64) * np.uint64(stride)
        sh = [1] * (len(inner) + 1)
        sh[d] = m
        idx = idx + ar.reshape(sh)
        stride *= m
    z = np.asarray(zidx, dtype=np.uint64) * np.uint64(stride)
    idx = idx + z.reshape([1] * len(inner) + [len(zidx)])
    return hash_values(idx, seed, dtype)


def equal_bits(a, b):
    """Bitwise equality treating every NaN as equal (NaN payloads differ by CPU/GPU)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    both_nan = np.isnan(a) & np.isnan(b)
    ui = np.uint32 if a.dtype == np.float32 else np.uint64
    same = a.view(ui) == b.view(ui)
    return bool(np.all(same | both_nan))


def first_mismatch(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    ui = np.uint32 if a.dtype == np.float32 else np.uint64
    bad = (a.view(ui) != b.view(ui)) & ~(np.isnan(a) & np.isnan(b))
    idx = np.argwhere(bad)
    if len(idx) == 0:
        return None
    i = tuple(idx[0])
    return i, a[i], b[i], int(bad.sum())


def gpts(points, seconds):
    return points / seconds / 1e9 if seconds > 0 else math.inf


# ---------------------------------------------------------------------------
# The CPU baseline leg of bench.py: the reference's vectorised launch
# (runtime.py:596-618 via run_body) over one image, split along the slowest axis
# across host threads (numpy releases the GIL inside ufunc loops).


def threaded_machine_step(blk, lo, hi, kir, scalars=None, dtype=np.float64, pool=None, nthreads=1):
    """One ``HALO_TRANSFER`` + full-interior launch on padded block ``blk`` (in place).

    The launch range is cut into tiles of about 128K points along the block's two
    slowest-varying memory axes, so every thread's numpy temporaries stay in its
    cache; each tile is one ``_launch_vector`` over its sub-range (the arithmetic is
    ``run_body``'s, unchanged, and tiles write disjoint cells of the live buffer
    while reading the snapshot).  The snapshot copy (runtime.py:596) is split the
    same way across the threads.
    """
    halo_fill(blk, lo, hi)
    shape = tuple(s - a - b for s, a, b in zip(blk.shape, lo, hi))
    nd = blk.ndim
    # memory axes from slowest to fastest
    order = list(range(nd)) if blk.flags.c_contiguous else list(range(nd - 1, -1, -1))
    snap = np.empty_like(blk)
    ax0 = order[0]
    nslow = blk.shape[ax0]
    step0 = max(1, nslow // max(1, 4 * nthreads))

    def copy(z0):
        idx = [slice(None)] * nd
        idx[ax0] = slice(z0, min(nslow, z0 + step0))
        snap[tuple(idx)] = blk[tuple(idx)]

    if pool is None or nthreads <= 1:
        snap[...] = blk
    else:
        list(pool.map(copy, range(0, nslow, step0)))
    # tiles of ~128K points: the fast axes whole, the slowest axis cut, and the next one
    # too when one index of the slowest axis already holds more than that
    target = 1 << 17

    def cuts(n, c):
        return [(z, min(n, z + c - 1)) for z in range(1, n + 1, c)]

    ax_s = order[0]
    inner = int(np.prod([shape[d] for d in order[1:]])) if nd > 1 else 1
    tiles = []
    for rs in cuts(shape[ax_s], max(1, target // inner)):
        if nd > 2 and inner > target:
            ax_t = order[1]
            for rt in cuts(shape[ax_t], max(1, target // (inner // shape[ax_t]))):
                t = [(1, m) for m in shape]
                t[ax_s], t[ax_t] = rs, rt
                tiles.append(t)
        else:
            t = [(1, m) for m in shape]
            t[ax_s] = rs
            tiles.append(t)
    name = kir.array_params[0]

    def work(ranges):
        def read(_name, offsets):
            return snap[tuple(slice(a - 1 + h + o, e + h + o)
                              for (a, e), h, o in zip(ranges, lo, offsets))]

        pending = run_body(kir, read, scalars, dtype)
        blk[tuple(slice(a - 1 + h, e + h) for (a, e), h in zip(ranges, lo))] = pending[name]

    if pool is None or nthreads <= 1:
        for t in tiles:
            work(t)
    else:
        list(pool.map(work, tiles))
    return blk
