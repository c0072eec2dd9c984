"""Commit-ready SASS evidence: NVRTC-compile the benchmark kernels (no GPU needed), write
each kernel family's full SASS listing under OUT/, and a summary of the instructions
that show the design: TMA loads (UTMALDG), mbarrier traffic (SYNCS), 16-byte global
stores (STG.E.128), 16-byte shared loads (LDS.128), paired fp32 adds (FADD2), fp64 adds,
and the absence of contracted FMAs in division-free kernels.
    python tools/sass_excerpts.py profiles/r02/sass"""
import collections
import json
import pathlib
import re
import shutil
import subprocess
import sys
import tempfile

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

from paper_1502_03504_b200 import _lib, stencils  # noqa: E402
from paper_1502_03504_b200.ir import KernelBuilder, serialize  # noqa: E402

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
KEYS = ("UTMALDG", "SYNCS", "STG.E.128", "STG.E", "LDS.128", "LDG.E.128", "FADD2", "FADD", "FMUL", "DADD",
        "DFMA", "FFMA", "FFMA2", "SHFL", "NANOSLEEP")


def two3d():
    kb = KernelBuilder("two3d", 3)
    u, v = kb.array("u"), kb.array("v")
    kb.store(u, u[0, 0, 0] + 0.125 * (u[-1, 0, 0] + u[1, 0, 0] + u[0, -1, 0] + u[0, 1, 0]
                                      + u[0, 0, -1] + u[0, 0, 1] - 6 * u[0, 0, 0]) + 0.5 * v[0, 0, 0])
    return kb.build()


CASES = [("lap3d7", "f32", stencils.lap3d7, ("lope_tiled",)),
         ("box5x5", "f64", stencils.box5x5, ("lope_tiled",)),
         ("ninept2d", "f32", stencils.ninept2d, ("lope_tiled",)),
         ("heat2d", "f32", stencils.heat2d, ("lope_tblock", "lope_tiled")),
         ("two3d", "f32", two3d, ("lope_tiled_multi",)),
         ("avg3", "f64", stencils.avg3, ("lope_row",))]


def opcode(line):
    m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    return m.group(2) if m else None


def main():
    out = pathlib.Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/sass")
    out.mkdir(parents=True, exist_ok=True)
    summary = {}
    for name, dt, make, funs in CASES:
        tmp = tempfile.mkdtemp()
        try:
            _lib.lib().lope_set_cache_dir(tmp.encode())
            h = _lib.compile_kernel(serialize(make()), dt)
            _lib.destroy_kernel(h)
            cubin = next(pathlib.Path(tmp).glob("*.cubin"))
            for fun in funs:
                sass = subprocess.run([CUOBJDUMP, "-sass", "-fun", fun, str(cubin)],
                                      capture_output=True, text=True).stdout
                res = subprocess.run([CUOBJDUMP, "-res-usage", str(cubin)], capture_output=True, text=True).stdout
                (out / f"{name}_{dt}_{fun}.sass").write_text(sass)
                c = collections.Counter()
                n = 0
                for line in sass.splitlines():
                    op = opcode(line)
                    if not op:
                        continue
                    n += 1
                    for k in KEYS:
                        if op == k or op.startswith(k + "."):
                            c[k] += 1
                usage = ""
                lines = res.splitlines()
                for i, line in enumerate(lines):
                    if f"Function {fun}:" in line and i + 1 < len(lines):
                        usage = lines[i + 1].strip()
                summary[f"{name}:{dt}:{fun}"] = {"static_instructions": n, "resources": usage,
                                                 "opcodes": {k: c[k] for k in KEYS if c[k]}}
        finally:
            _lib.lib().lope_set_cache_dir(str(_lib.CACHE_DIR).encode())
            shutil.rmtree(tmp, ignore_errors=True)
    (out / "summary.json").write_text(json.dumps(summary, indent=1))
    for k, v in summary.items():
        print(k, v["static_instructions"], v["resources"][:60], v["opcodes"])


if __name__ == "__main__":
    main()
