"""GPU fuzz: random locally-oriented kernels through the product path vs the oracle.

Random IR trees (+ - * / with constant, scalar and expression divisors, abs, sqrt,
min, max, locals, pending-centre reads, one or two arrays), random rank 1/2/3, halos at
least the footprint (sometimes wider, asymmetric), ragged or vector-aligned shapes,
fp32 and fp64; ``iterate`` (one array) or ``iterate_arrays`` / per-step launches (two
arrays) for a few steps (tiled, RAG, row, multi-array or temporal-blocking kernels,
fused halo images) compared bit for bit with the numpy restatement (fp64 == the
reference's arithmetic).  Prints the launches per kernel family.  Exits non-zero on a
mismatch.

    python tools/fuzz_gpu.py [cases] [seed] [--decomp]

``--decomp``: slab / fused-peer / grid decompositions on one GPU vs the undecomposed run.
"""

import pathlib
import random
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

from oracle import lope_oracle as O  # noqa: E402
from paper_1502_03504_b200 import runtime as R  # noqa: E402
from paper_1502_03504_b200.ir import KernelBuilder, fabs, fmax, fmin, fsqrt  # noqa: E402


def rand_expr(rng, depth, rank, arrays, scalars, locals_):
    if depth == 0 or rng.random() < 0.25:
        kind = rng.randrange(5)
        if kind <= 1:
            a = rng.choice(arrays)
            return a[tuple(rng.randrange(-2, 3) for _ in range(rank))]
        if kind == 2:
            return float(rng.choice([1, 2, 3, 0.5, 0.125, 1.5, 7, 0.1]))
        if kind == 3 and scalars:
            return rng.choice(scalars)
        if locals_:
            return rng.choice(locals_)
        return arrays[0][(0,) * rank]
    a = rand_expr(rng, depth - 1, rank, arrays, scalars, locals_)
    b = rand_expr(rng, depth - 1, rank, arrays, scalars, locals_)
    r = rng.random()
    if r < 0.08:
        return fabs(a)
    if r < 0.13:
        return fsqrt(fabs(a))
    if r < 0.19:
        return fmin(a, b)
    if r < 0.25:
        return fmax(a, b, rand_expr(rng, 0, rank, arrays, scalars, locals_))
    if r < 0.33:
        return a / rng.choice([3.0, 7.0, 25.0, 0.1, 2.0]) if rng.random() < 0.7 else a / (fabs(b) + 1.0)
    if r < 0.40 and scalars:
        return a / scalars[0]
    op = rng.choice(["+", "-", "*"])
    return a + b if op == "+" else (a - b if op == "-" else a * b)


def make_kernel(rng, rank):
    kb = KernelBuilder("fz", rank)
    narr = 2 if rng.random() < 0.2 else 1
    arrays = [kb.array(n) for n in ("u", "v")[:narr]]
    scalars = [kb.scalar("c")] if rng.random() < 0.5 else []
    locals_ = []
    if rng.random() < 0.3:
        locals_.append(kb.let("t", rand_expr(rng, 2, rank, arrays, scalars, [])))
    kb.store(arrays[0], rand_expr(rng, 3, rank, arrays, scalars, locals_))
    if narr == 2 and rng.random() < 0.5:
        kb.store(arrays[1], rand_expr(rng, 2, rank, arrays, scalars, locals_) + arrays[0][(0,) * rank])
    return kb.build()


PATHS = {}


def run_case(rng, case):
    rank = rng.choice([1, 2, 2, 2, 3, 3])
    try:
        kir = make_kernel(rng, rank)
    except ValueError:          # E103-style programs the checker rejects
        return None
    dt = rng.choice(["float32", "float64"])
    npdt = np.float32 if dt == "float32" else np.float64
    vx = 4 if dt == "float32" else 2
    fps = [kir.footprints[a].dims for a in kir.array_params]
    lo = [max(f[d][0] for f in fps) + (rng.randrange(2) if rng.random() < 0.3 else 0) for d in range(rank)]
    hi = [max(f[d][1] for f in fps) + (rng.randrange(2) if rng.random() < 0.3 else 0) for d in range(rank)]
    if rank == 1:
        shape = (rng.choice([rng.randrange(max(lo[0] + hi[0], 2), 64), rng.randrange(64, 5000)]),)
    elif rank == 2:
        mx = rng.choice([rng.randrange(9, 90) * vx, rng.randrange(20, 300), 288, 320])
        shape = (mx, rng.randrange(max(lo[1] + hi[1], 5), 80))
    else:
        mx = rng.choice([rng.randrange(9, 40) * vx, rng.randrange(5, 160)])     # ragged x too
        shape = (mx, rng.randrange(max(lo[1] + hi[1], 4), 30),
                 rng.randrange(max(lo[2] + hi[2], 3), 20))
    if any(s < l + h or s < 1 for s, l, h in zip(shape, lo, hi)):
        return None
    sc = {"c": rng.choice([0.25, 3.0, -1.5, 7.0])} if "c" in kir.scalar_params else None
    steps = rng.randrange(1, 6)
    fields = [O.hash_field(shape, 100 + case + 7 * i, npdt) for i in range(len(kir.array_params))]
    k = R.CompiledKernel(kir, dt)
    arrs = []
    for f in fields:
        a = R.HaloArray(shape, lo, hi, dt)
        a.set_interior(f)
        arrs.append(a)
    if len(arrs) == 1:
        R.iterate(k, arrs[0], steps, sc)
        got = [arrs[0].get_interior()]
        want = fields[0]
        with np.errstate(all="ignore"):
            for _ in range(steps):
                want = np.broadcast_to(O.periodic_apply(want, kir, sc, npdt), shape).astype(npdt)
        want = [want]
    else:
        # two arrays: either one launch per step after a periodic halo fill of both, or
        # iterate_arrays (fused steps storing every stored array's images); the oracle
        # works on the dense periodic fields
        cur = list(fields)
        if rng.random() < 0.5:
            R.iterate_arrays(k, arrs, steps, sc)
        else:
            for _ in range(steps):
                for a in arrs:
                    R.halo_transfer(a)
                R.launch(k, arrs, None, sc)
        for _ in range(steps):
            with np.errstate(all="ignore"):
                cur = _oracle_multi(kir, cur, sc, npdt)
        got = [a.get_interior() for a in arrs]
        want = cur
    import json as _json
    for fam, n in _json.loads(k.describe())["launches"].items():
        PATHS[fam] = PATHS.get(fam, 0) + n
    for g_, w_ in zip(got, want):
        if not O.equal_bits(g_, w_):
            return (kir, dt, shape, lo, hi, steps, O.first_mismatch(g_, w_))
    return True


def run_decomp_case(rng, case):
    """One-array kernel, random slab count / grid: MultiSlab, PeerMultiSlab and MultiGrid
    against the undecomposed run (the multi-GPU orchestration with in-process images)."""
    from paper_1502_03504_b200 import dist as D
    rank = 2 if rng.random() < 0.6 else 3
    try:
        kb_kir = make_kernel(rng, rank)
    except ValueError:
        return None
    if len(kb_kir.array_params) != 1:
        return None
    kir = kb_kir
    dt = rng.choice(["float32", "float64"])
    npdt = np.float32 if dt == "float32" else np.float64
    vx = 4 if dt == "float32" else 2
    fp = kir.footprints[kir.array_params[0]].dims
    lo = [n for n, _ in fp]
    hi = [p for _, p in fp]
    P = rng.choice([2, 3, 4])
    mx = rng.randrange(9, 60) * vx if rng.random() < 0.5 else rng.randrange(max(lo[0] + hi[0], 5), 200)
    if rank == 2:
        shape = (mx, P * rng.randrange(max(lo[1] + hi[1], 3), 20))
    else:
        shape = (mx, rng.randrange(max(lo[1] + hi[1], 4), 24),
                 P * rng.randrange(max(lo[2] + hi[2], 3), 10))
    if any(s < l + h for s, l, h in zip(shape, lo, hi)):
        return None
    sc = {"c": rng.choice([0.25, 3.0, -1.5])} if "c" in kir.scalar_params else None
    steps = rng.randrange(2, 5)
    field = O.hash_field(shape, 500 + case, npdt)
    k = R.CompiledKernel(kir, dt)
    base = R.HaloArray(shape, lo, hi, dt)
    base.set_interior(field)
    R.iterate(k, base, steps, sc)
    want = base.get_interior()
    runs = [("slab", D.MultiSlab(k, shape, lo, hi, dt, P, sc)),
            ("peer", D.PeerMultiSlab(k, shape, lo, hi, dt, P, sc))]
    splits = [1] * rank
    splits[rng.randrange(rank)] = P
    if all(s % q == 0 for s, q in zip(shape, splits)) and all(
            s // q >= l + h or q == 1 for s, q, l, h in zip(shape, splits, lo, hi)):
        runs.append(("grid", D.MultiGrid(k, D.CartGrid(shape, splits, lo, hi), dt, sc)))
    for name, ms in runs:
        ms.set_global(field)
        ms.iterate(steps)
        got = ms.get_global()
        if not O.equal_bits(got, want):
            return (kir, dt, shape, lo, hi, steps, (name, P, splits, O.first_mismatch(got, want)))
    return True


def _oracle_multi(kir, fields, sc, npdt):
    axes = tuple(range(fields[0].ndim))
    names = list(kir.array_params)

    def read(name, offsets):
        f = fields[names.index(name)]
        if all(o == 0 for o in offsets):
            return f.copy()
        return np.roll(f, shift=tuple(-o for o in offsets), axis=axes)

    pending = O.run_body(kir, read, sc, npdt)
    return [np.broadcast_to(np.asarray(pending[n], dtype=npdt), fields[0].shape).copy() if n in pending
            else fields[i] for i, n in enumerate(names)]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cases = int(args[0]) if len(args) > 0 else 200
    seed = int(args[1]) if len(args) > 1 else 1
    rng = random.Random(seed)
    decomp = "--decomp" in sys.argv
    ran = bad = 0
    for c in range(cases):
        r = run_decomp_case(rng, c) if decomp else run_case(rng, c)
        if r is None:
            continue
        ran += 1
        if r is not True:
            bad += 1
            kir, dt, shape, lo, hi, steps, mm = r
            print("MISMATCH", dt, shape, lo, hi, steps, mm, kir, flush=True)
    print(f"fuzz: {ran} cases, {bad} mismatches", flush=True)
    if PATHS:
        print("launches per kernel family:", PATHS, flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
