"""Debug: NVRTC-compile one kernel under LOPE_TILE/LOPE_MB/LOPE_PW overrides (no GPU needed)
and print the tiled kernel's register / stack usage from cuobjdump."""
import os, sys, pathlib, subprocess, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1502_03504_b200 import _lib, stencils
from paper_1502_03504_b200.ir import serialize
name, dt = sys.argv[1], sys.argv[2]
import tempfile
tmp = tempfile.mkdtemp()
_lib.lib().lope_set_cache_dir(tmp.encode())
k = _lib.compile_kernel(serialize(stencils.by_name(name)), dt)
_lib.destroy_kernel(k)
f = next(pathlib.Path(tmp).glob("*.cubin"))
out = subprocess.run(["cuobjdump", "-res-usage", str(f)], capture_output=True, text=True).stdout
lines = out.splitlines()
for i, line in enumerate(lines):
    if "lope_tiled" in line and i + 1 < len(lines):
        print(os.environ.get("LOPE_TILE"), os.environ.get("LOPE_MB"), lines[i + 1].strip()[:90])
sass = subprocess.run(["cuobjdump", "-sass", "-fun", "lope_tiled", str(f)], capture_output=True, text=True).stdout
import collections
c = collections.Counter()
for line in sass.splitlines():
    for op in ("LDL", "STL", "CALL", "DFMA", "DADD", "DMUL", "MUFU.RCP64H", "FFMA", "FADD"):
        if f" {op}" in line:
            c[op] += 1
print("  static SASS counts:", dict(c))
