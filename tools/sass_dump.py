"""NVRTC-compile one stencil (no GPU needed) under the LOPE_* tile overrides and write the
SASS of one of its kernels (default lope_tiled) to stdout, with an opcode histogram on stderr.
    python tools/sass_dump.py lap3d7 f32 [kernel]"""
import collections, os, pathlib, subprocess, sys, tempfile
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1502_03504_b200 import _lib, stencils
from paper_1502_03504_b200.ir import serialize

name, dt = sys.argv[1], sys.argv[2]
fun = sys.argv[3] if len(sys.argv) > 3 else "lope_tiled"
tmp = tempfile.mkdtemp()
_lib.lib().lope_set_cache_dir(tmp.encode())
k = _lib.compile_kernel(serialize(stencils.by_name(name)), dt)
_lib.destroy_kernel(k)
f = next(pathlib.Path(tmp).glob("*.cubin"))
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fun, str(f)], capture_output=True, text=True).stdout
print(sass)
c = collections.Counter()
for line in sass.splitlines():
    parts = line.split("*/")
    if len(parts) < 2 or "/*" not in line:
        continue
    ins = parts[1].strip().rstrip(";").strip()
    if not ins or ins.startswith("/*"):
        continue
    toks = ins.split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    c[op.split(".")[0]] += 1
print(sum(c.values()), "static instructions:", dict(c.most_common(30)), file=sys.stderr)
