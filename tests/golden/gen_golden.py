"""Generate the golden fixtures from the reference implementation itself.

Run in the build container (the only place ``/root/reference`` exists)::

    python tests/golden/gen_golden.py

It imports the read-only reference package ``lopec`` (``/root/reference/pkg/src``),
compiles ``.lope`` programs with the reference frontend, runs them on the
reference ``Machine`` / ``oracle_step`` in float64 and writes small fixtures:

* ``kernels.json``  — every kernel's reference lowering, serialised in this
  repo's LOPE1 text form (pins ``stencils.py`` and the IR converter);
* ``runs.npz``      — input fields and reference outputs for K = 1/5/20 steps,
  single image and slab-decomposed (``images=P, grid_rows=P``), plus rank-3
  ``oracle_step`` runs;
* ``exchange.npz``  — every padded cell of every block after one
  ``HALO_TRANSFER`` on slab-decomposed grids (``runtime.py:643-711``);
* ``random.npz`` + ``random.json`` — random kernels (offsets in [-2,2], + - * /,
  abs/min/max/sqrt, scalar parameters, locals) with one ``oracle_step``;
* ``kats.json``     — point-source / corner / fixed-point / layout KATs;
* ``config_digests.json`` (``--configs``) — SHA-256 of the reference ``Machine``'s
  fp64 output at the exact BASELINE sizes it can run (configs 1, 2 and 4, the last
  one slab-decomposed over 8 images).

Nothing here runs on the GPU box; the fixtures travel, the reference does not.
"""

from __future__ import annotations

import json
import os
import pathlib
import random
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.dont_write_bytecode = True

from lopec import check_program, parse_source  # noqa: E402
from lopec.ir import StorageLayout, lower_kernel, map_local_to_global  # noqa: E402
from lopec.runtime import Machine, RunConfig, oracle_step  # noqa: E402

from paper_1502_03504_b200.ir import from_lopec, serialize  # noqa: E402

CORPUS = pathlib.Path("/root/reference/pkg/corpus")

from oracle.lope_programs import KERNEL_SRC, MAIN_2D, program_text  # noqa: E402


def compile_text(text, name="gen.lope"):
    program, diags = parse_source(text, name)
    assert program is not None and not diags, [d.render() for d in diags]
    result = check_program(program)
    assert result.ok, [d.render() for d in result.diagnostics]
    return result


def program_for(kname):
    return compile_text(program_text(kname))


def run_machine(result, field, **kw):
    m = Machine(result, RunConfig(**kw), field)
    m.run()
    return m


def gen_kernels():
    out = {}
    for stem, kname in (("laplacian", "laplacian"), ("avg3", "avg3"), ("upwind", "drift2")):
        r = compile_text((CORPUS / f"{stem}.lope").read_text(), f"{stem}.lope")
        out[kname] = serialize(from_lopec(lower_kernel(r.kernels[kname])))
    for kname in KERNEL_SRC:
        r = program_for(kname)
        out[kname] = serialize(from_lopec(lower_kernel(r.kernels[kname])))
    (HERE / "kernels.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    return out


def gen_runs():
    rng = np.random.default_rng(20260823)     # seed of test_acceptance.py:91
    arrays = {}
    index = []
    cases = [
        ("laplacian", CORPUS / "laplacian.lope", (8, 8), {}),
        ("laplacian", CORPUS / "laplacian.lope", (32, 32), {}),
        ("avg3", CORPUS / "avg3.lope", (64, 1), {}),
        ("drift2", CORPUS / "upwind.lope", (32, 32), {"c": 0.25}),
        ("heat2d", None, (32, 24), {}),
        ("ninept2d", None, (24, 32), {}),
        ("box5x5", None, (20, 16), {}),
    ]
    for kname, path, shape, scal in cases:
        result = (compile_text(path.read_text(), path.name) if path is not None
                  else program_for(kname))
        kir = lower_kernel(result.kernels[kname])
        for steps in (1, 5, 20):
            field = rng.uniform(-1.0, 1.0, shape)
            tag = f"{kname}_{shape[0]}x{shape[1]}_k{steps}"
            base = run_machine(result, field.copy(), images=1, steps=steps).gather()
            ref = field[:, 0] if shape[1] == 1 else field.copy()
            for _ in range(steps):
                ref = oracle_step(ref, kir, {k: np.float64(v) for k, v in scal.items()})
            got = base[:, 0] if shape[1] == 1 else base
            assert np.array_equal(ref, got), tag
            arrays[tag + "_in"] = field[:, 0] if shape[1] == 1 else field
            arrays[tag + "_out"] = got
            decomp = []
            if shape[1] > 1:
                for p in (2, 4):
                    if shape[1] % p == 0 and shape[1] // p >= max(1, KERNEL_SRC.get(kname, ("", 2, 2))[2]):
                        g = run_machine(result, field.copy(), images=p, grid_rows=p,
                                        steps=steps).gather()
                        assert np.array_equal(g, base), (tag, p)
                        decomp.append(p)
            index.append({"tag": tag, "kernel": kname, "shape": list(got.shape), "steps": steps,
                          "scalars": scal, "decomp_checked": decomp})
    # rank 3: the reference Machine rejects rank-3 coarrays (F6); oracle_step covers it
    result = program_for("lap3d7")
    kir = lower_kernel(result.kernels["lap3d7"])
    for shape, steps in (((12, 10, 8), 1), ((12, 10, 8), 5), ((9, 7, 6), 20)):
        field = rng.uniform(-1.0, 1.0, shape)
        ref = field.copy()
        for _ in range(steps):
            ref = oracle_step(ref, kir, {})
        tag = f"lap3d7_{'x'.join(map(str, shape))}_k{steps}"
        arrays[tag + "_in"] = field
        arrays[tag + "_out"] = ref
        index.append({"tag": tag, "kernel": "lap3d7", "shape": list(shape), "steps": steps,
                      "scalars": {}, "decomp_checked": []})
    np.savez_compressed(HERE / "runs.npz", **arrays)
    (HERE / "runs.json").write_text(json.dumps(index, indent=1) + "\n")


EXCHANGE_TEMPLATE = """\
program main
  real, allocatable, dimension(:,:), codimension[:,:], &
        HALO({l0}:*:{h0}, {l1}:*:{h1}) :: U
  allocate(U(1-{l0}:M+{h0}, 1-{l1}:N+{h1})[MP,*])
  call HALO_TRANSFER(U, BC=CYCLIC)
end program main
"""


def gen_exchange():
    rng = np.random.default_rng(104)
    arrays = {}
    index = []
    for widths in ((1, 1, 1, 1), (2, 2, 2, 2), (2, 0, 1, 1), (0, 2, 2, 1), (1, 2, 0, 0)):
        result = compile_text(EXCHANGE_TEMPLATE.format(l0=widths[0], h0=widths[1],
                                                       l1=widths[2], h1=widths[3]))
        for p in (1, 2, 4):
            field = rng.uniform(-1, 1, (8, 8))
            m = run_machine(result, field.copy(), images=p, grid_rows=p)
            tag = f"x{''.join(map(str, widths))}_p{p}"
            arrays[tag + "_in"] = field
            for k in m.images:
                arrays[f"{tag}_blk{k}"] = m.arrays["u"].view(k).copy()
            index.append({"tag": tag, "widths": list(widths), "p": p})
    np.savez_compressed(HERE / "exchange.npz", **arrays)
    (HERE / "exchange.json").write_text(json.dumps(index, indent=1) + "\n")


def _rand_expr(rng, depth, rank, scalars):
    if depth == 0 or rng.random() < 0.3:
        kind = rng.randrange(4 if scalars else 3)
        if kind == 0:
            offs = [rng.randrange(-2, 3) for _ in range(rank)]
            return "U(" + ",".join(("+" if o > 0 else "") + str(o) for o in offs) + ")"
        if kind == 1:
            return f"{rng.randrange(1, 5)}"
        if kind == 2:
            return f"{rng.uniform(0.25, 2.0):.3f}"
        return rng.choice(scalars)
    r = rng.random()
    a = _rand_expr(rng, depth - 1, rank, scalars)
    b = _rand_expr(rng, depth - 1, rank, scalars)
    if r < 0.12:
        return f"abs({a})"
    if r < 0.20:
        return f"sqrt(abs({a}))"
    if r < 0.27:
        return f"min({a}, {b})"
    if r < 0.34:
        return f"max({a}, {b}, {_rand_expr(rng, 0, rank, scalars)})"
    op = rng.choice(["+", "-", "*", "/"])
    return f"({a} {op} {b})"


def gen_random():
    rng = random.Random(20260823)
    nrng = np.random.default_rng(12)
    arrays = {}
    meta = []
    trial = -1
    attempt = 0
    while len(meta) < 60:
        attempt += 1
        n = len(meta)
        rank = 2 if n < 40 else (3 if n < 52 else 1)
        trial = n
        if attempt > 100000:
            raise RuntimeError("random kernel generation did not converge")
        use_scalars = trial % 3 == 0
        scal_names = ["c", "q"] if use_scalars else []
        body = ""
        decls = ""
        if use_scalars:
            decls += "  real :: c\n  integer :: q\n"
        if trial % 4 == 1:
            decls += "  real :: t\n"
            body += "  t = " + _rand_expr(rng, 2, rank, scal_names) + "\n"
            scal_names = scal_names + ["t"]
        body += ("  U(" + ",".join(["0"] * rank) + ") = "
                 + _rand_expr(rng, 3, rank, scal_names) + "\n")
        if trial % 5 == 2:
            body += ("  U(" + ",".join(["0"] * rank) + ") = U(" + ",".join(["0"] * rank)
                     + ") * 0.5 + " + f"{rng.uniform(0.25, 2.0):.3f}" + "\n")
        dims = ",".join([":"] * rank)
        halo = ", ".join(["2:*:2"] * rank)
        params = "U" + (", c, q" if use_scalars else "")
        text = (f"pure concurrent subroutine k({params})\n"
                f"  real, dimension({dims}), HALO({halo}) :: U\n{decls}{body}"
                f"end subroutine k\n\nprogram main\nend program main\n")
        result = compile_text(text)
        kir = lower_kernel(result.kernels["k"])
        # keep only kernels whose stored value depends on the field at >= 2 offsets
        n_reads = sum(repr(st.expr).count("Read(") for st in kir.body)
        if n_reads < 2 or all(o == 0 for fp in kir.footprints.values() for d in fp.dims for o in d):
            continue
        shape = {1: (11,), 2: (9, 7), 3: (7, 6, 5)}[rank]
        field = nrng.uniform(-1, 1, shape)
        scal = {"c": np.float64(0.75), "q": np.int64(3)} if use_scalars else {}
        with np.errstate(all="ignore"):
            out = oracle_step(field, kir, scal)
        arrays[f"r{trial}_in"] = field
        arrays[f"r{trial}_out"] = out
        meta.append({"trial": trial, "rank": rank, "source": text,
                     "ir": serialize(from_lopec(kir)),
                     "scalars": {"c": 0.75, "q": 3} if use_scalars else {}})
    np.savez_compressed(HERE / "random.npz", **arrays)
    (HERE / "random.json").write_text(json.dumps(meta, indent=1) + "\n")


def gen_kats():
    lap = compile_text((CORPUS / "laplacian.lope").read_text(), "laplacian.lope")
    kats = {}
    f = np.zeros((4, 4)); f[1, 1] = 1.0
    kats["point_source"] = run_machine(lap, f, images=1, steps=1).gather().tolist()
    f = np.zeros((4, 4)); f[0, 0] = 1.0
    kats["corner_source"] = run_machine(lap, f, images=1, steps=1).gather().tolist()
    f = np.full((8, 8), 1.0)
    kats["fixed_point_ones_25"] = bool(np.array_equal(
        run_machine(lap, f.copy(), images=1, steps=25).gather(), f))
    lay = StorageLayout((8, 4), (1, 1), (1, 1))
    kats["layout_12"] = map_local_to_global((1, 0), (1, 1), lay)
    kats["layout_59"] = map_local_to_global((1, 1), (8, 4), lay)
    # sub-range launch: only i=2:M-1, j=3:N updated, the rest copied through
    sub = compile_text("""\
pure concurrent subroutine k(U)
  real, dimension(:,:), HALO(1:*:1, 1:*:1) :: U
  U(0,0) = U(0,0)*0.5 + U(-1,0) - U(0,+1)*0.25
end subroutine k

program main
  real, allocatable, dimension(:,:), codimension[:,:], HALO(1:*:1,1:*:1) :: U
  integer :: device
  integer :: it
  device = GET_SUBIMAGE(1)
  allocate(U(0:M+1, 0:N+1)[MP,*])
  do it = 1, nsteps
    call HALO_TRANSFER(U, BC=CYCLIC)
    do concurrent (i=2:M-1, j=3:N) [[device]]
      call k( U(i,j)[device] )
    end do
  end do
end program main
""")
    rng = np.random.default_rng(55)
    f = rng.uniform(-1, 1, (10, 9))
    m = run_machine(sub, f.copy(), images=1, steps=3)
    kats["subrange_in"] = f.tolist()
    kats["subrange_out_padded"] = m.arrays["u"].view(1).tolist()
    kats["subrange_ir"] = serialize(from_lopec(lower_kernel(sub.kernels["k"])))
    twice = compile_text("""\
pure concurrent subroutine twice(U)
  real, dimension(:,:), HALO(1:*:1, 1:*:1) :: U
  U(0,0) = U(0,0)*2
  U(0,0) = U(0,0) + 1
end subroutine twice

program main
end program main
""")
    kats["twice_ir"] = serialize(from_lopec(lower_kernel(twice.kernels["twice"])))
    # two-array kernel: reads V at offsets, stores U and V (pending centre of U)
    two = compile_text("""\
pure concurrent subroutine mix(U, V)
  real, dimension(:,:), HALO(1:*:1, 1:*:1) :: U
  real, dimension(:,:), HALO(1:*:1, 1:*:1) :: V
  U(0,0) = U(0,0) + 0.5*V(-1,0) - V(0,+1)
  V(0,0) = V(0,0)*0.25 + U(0,0)
end subroutine mix

program main
  real, allocatable, dimension(:,:), codimension[:,:], HALO(1:*:1,1:*:1) :: U
  real, allocatable, dimension(:,:), codimension[:,:], HALO(1:*:1,1:*:1) :: V
  integer :: device
  integer :: it
  device = GET_SUBIMAGE(1)
  allocate(U(0:M+1, 0:N+1)[MP,*])
  allocate(V(0:M+1, 0:N+1)[MP,*])
  V(:,:) = U(:,:)
  do it = 1, nsteps
    call HALO_TRANSFER(U, BC=CYCLIC)
    call HALO_TRANSFER(V, BC=CYCLIC)
    do concurrent (i=1:M, j=1:N) [[device]]
      call mix( U(i,j)[device], V(i,j)[device] )
    end do
  end do
end program main
""")
    f = rng.uniform(-1, 1, (8, 6))
    m = run_machine(two, f.copy(), images=1, steps=4)
    kats["mix_in"] = f.tolist()
    kats["mix_out_u"] = m.arrays["u"].view(1).tolist()
    kats["mix_out_v"] = m.arrays["v"].view(1).tolist()
    kats["mix_ir"] = serialize(from_lopec(lower_kernel(two.kernels["mix"])))
    (HERE / "kats.json").write_text(json.dumps(kats, indent=1) + "\n")


# Programs for the Machine drop-in tests: written here (not copied from the corpus),
# each with a device subimage so the mirror path and its counters are exercised.
MACHINE_MAIN = """\
{kernel}
program main
  real, allocatable, dimension({dims}), codimension[{codims}], HALO({halo}) :: U
  integer :: device
  integer :: it
  device = GET_SUBIMAGE({sub})
  allocate(U({bounds})[{cob}])
  if (device /= this_image()) then
    allocate(U[device], HALO_SRC=U) [[device]]
  end if
  do it = 1, nsteps
    call HALO_TRANSFER(U, BC=CYCLIC)
    do concurrent ({conc}) [[device]]
      call {kname}( U({idx})[device]{extra} )
    end do
  end do
  if (device /= this_image()) then
    U = U[device]
  end if
end program main
"""

MACHINE_KERNELS = {
    "fig1": ("""\
pure concurrent subroutine fig1(U)
  real, dimension(:,:), HALO(:,:) :: U
  U(0,0) = U(0,+1) + U(-1,0) - 3*U(0,0) + U(+1,0) + U(0,-1)
end subroutine fig1
""", 2, (1, 1, 1, 1), ""),
    "mean3": ("""\
pure concurrent subroutine mean3(A)
  real, dimension(:), HALO(:) :: A
  A(0) = (A(-1) + A(0) + A(+1)) / 3
end subroutine mean3
""", 1, (1, 1), ""),
    "skew": ("""\
pure concurrent subroutine skew(U, c)
  real, dimension(:,:), HALO(:,:) :: U
  real :: c
  real :: t
  t = U(-1,0) - U(-2,0)
  U(0,0) = U(0,0) + c*t + 0.125*(U(0,-1) - 2*U(0,0) + U(0,+1))
end subroutine skew
""", 2, (2, 0, 1, 1), ", 0.25"),
}


def machine_program(kname, sub=1):
    src, rank, w, extra = MACHINE_KERNELS[kname]
    if rank == 1:
        l0, h0 = w
        return MACHINE_MAIN.format(kernel=src, dims=":", codims=":", halo=f"{l0}:*:{h0}", sub=sub,
                                   bounds=f"{1 - l0}:M+{h0}", cob="*", conc="i=1:M", kname=kname,
                                   idx="i", extra=extra)
    l0, h0, l1, h1 = w
    return MACHINE_MAIN.format(kernel=src, dims=":,:", codims=":,:", halo=f"{l0}:*:{h0}, {l1}:*:{h1}",
                               sub=sub, bounds=f"{1 - l0}:M+{h0}, {1 - l1}:N+{h1}", cob="MP,*",
                               conc="i=1:M, j=1:N", kname=kname, idx="i,j", extra=extra)


def gen_machine():
    rng = np.random.default_rng(777)
    cases = []
    arrays = {}
    for kname, shape, runs in (
            ("fig1", (8, 8), [(1, 1, 0, 3), (2, 1, 0, 3), (4, 2, 1, 2), (2, 2, 1, 2), (1, 1, 1, 1)]),
            ("mean3", (24, 1), [(1, 1, 0, 4), (4, 1, 1, 3)]),
            ("skew", (12, 8), [(1, 1, 1, 3), (2, 2, 0, 2), (4, 4, 1, 2)])):
        text = machine_program(kname)
        result = compile_text(text)
        field = rng.uniform(-1, 1, shape)
        for images, rows, devices, steps in runs:
            m = run_machine(result, field.copy(), images=images, grid_rows=rows, devices=devices, steps=steps)
            tag = f"{kname}_p{images}_r{rows}_d{devices}_k{steps}"
            arrays[tag + "_in"] = field
            arrays[tag + "_out"] = m.gather()
            for k in m.images:
                arrays[f"{tag}_blk{k}"] = m.arrays["u"].view(k).copy()
            cases.append({"tag": tag, "kernel": kname, "images": images, "grid_rows": rows,
                          "devices": devices, "steps": steps, "text": text,
                          "counters": {str(k): v for k, v in m.counters.items()},
                          "events": [list(e) for e in m.events]})
    np.savez_compressed(HERE / "machine.npz", **arrays)
    (HERE / "machine.json").write_text(json.dumps(cases, indent=1) + "\n")


def column_major_digest(a):
    """SHA-256 of an array's values in column-major (reference block) order."""
    import hashlib
    f = np.asfortranarray(a)
    return hashlib.sha256(memoryview(f.T)).hexdigest()


def hash_field_chunked(shape, seed, chunk=1024):
    """oracle.hash_field(shape, seed, float64) built a few planes at a time (bounded memory)."""
    from oracle.lope_oracle import hash_planes
    out = np.empty(shape, dtype=np.float64, order="F")
    n = shape[-1]
    for z0 in range(0, n, chunk):
        z1 = min(n, z0 + chunk)
        out[..., z0:z1] = hash_planes(shape, seed, np.arange(z0, z1), np.float64)
    return out


# BASELINE configurations the reference Machine itself can run (rank 2; fp64, its only
# precision), at their exact sizes; the input is the device hash field (seed 20260823).
CONFIG_RUNS = (
    # tag, kernel, shape, steps, images, grid_rows
    ("c1", "heat2d", (1024, 1024), 100, 1, 1),
    ("c1_p4", "heat2d", (1024, 1024), 100, 4, 4),
    ("c2", "ninept2d", (16384, 16384), 1, 1, 1),
    ("c4_p8", "box5x5", (32768, 32768), 1, 8, 8),
)


def gen_config_digests(only=None):
    """SHA-256 digests of the reference Machine's output at the BASELINE config sizes
    (runtime.py:308-337 via Machine.run / gather), for the full-size GPU parity tests.
    Too large to commit as arrays; the digest and a few sampled values travel."""
    import time
    path = HERE / "config_digests.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for tag, kname, shape, steps, images, rows in CONFIG_RUNS:
        if only and tag not in only:
            continue
        t0 = time.time()
        field = hash_field_chunked(shape, 20260823)
        result = program_for(kname)
        m = run_machine(result, field, images=images, grid_rows=rows, steps=steps)
        del field
        got = m.gather()
        del m
        samples = [[int(i), int(j), float(got[i, j])]
                   for i, j in ((0, 0), (shape[0] - 1, shape[1] - 1), (shape[0] // 2, shape[1] // 3),
                                (1, shape[1] - 2))]
        out[tag] = {"kernel": kname, "shape": list(shape), "dtype": "float64", "steps": steps,
                    "seed": 20260823, "images": images, "grid_rows": rows,
                    "sha256_column_major": column_major_digest(got), "samples": samples,
                    "seconds": round(time.time() - t0, 1)}
        del got
        print(tag, out[tag]["sha256_column_major"], out[tag]["seconds"], "s", flush=True)
        path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if "--configs" in sys.argv:
        gen_config_digests([a for a in sys.argv[2:]] or None)
        sys.exit(0)
    gen_kernels()
    gen_runs()
    gen_exchange()
    gen_random()
    gen_kats()
    gen_machine()
    for p in sorted(HERE.iterdir()):
        print(p.name, p.stat().st_size)
