"""Debug: time lope_step on the c3 workload under different tile/zchunk/grid settings."""
import os, sys, pathlib, subprocess, json
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
if os.environ.get("TUNE") != "1":
    os.environ["LOPE_AUTOTUNE"] = "0"      # env overrides below are the experiment
import torch
from paper_1502_03504_b200 import runtime as R, stencils
shape = tuple(int(x) for x in os.environ.get("SHAPE", "1024,1024,1024").split(","))
name = os.environ.get("KERNEL", "lap3d7")
dt = os.environ.get("DT", "float32")
if name == "copy3d":
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder("copy3d", 3); u = kb.array("u"); kb.store(u, u[0, 0, 0]); kir = kb.build()
elif name == "copy3dh":
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder("copy3dh", 3); u = kb.array("u"); kb.store(u, u[0, 0, 0] + 0 * (u[1, 1, 0] + u[-1, -1, 0])); kir = kb.build()
elif name == "copy2dh":
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder("copy2dh", 2); u = kb.array("u"); kb.store(u, u[0, 0] + 0 * (u[1, 1] + u[-1, -1])); kir = kb.build()
elif name == "copy3dz":
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder("copy3dz", 3); u = kb.array("u"); kb.store(u, u[0, 0, 0] + 0 * (u[0, 0, 1] + u[0, 0, -1])); kir = kb.build()
elif name in ("box5x5m", "box5x5s"):
    from paper_1502_03504_b200.ir import KernelBuilder
    kb = KernelBuilder(name, 2); u = kb.array("u"); acc = None
    for j in range(-2, 3):
        for i in range(-2, 3):
            acc = u[i, j] if acc is None else acc + u[i, j]
    kb.store(u, acc * 0.04 if name == "box5x5m" else acc); kir = kb.build()
else:
    kir = stencils.by_name(name)
k = R.CompiledKernel(kir, dt)
fp = kir.footprints[kir.array_params[0]].dims
a = R.HaloArray(shape, [n for n, _ in fp], [p for _, p in fp], dt)
a.fill_hash(1)
_gap = None
if os.environ.get("GAP_GB"):
    _gap = torch.empty(int(float(os.environ["GAP_GB"]) * (1 << 30)), dtype=torch.uint8, device="cuda")
a.spare()
print("in/out buffer addresses", hex(a.data.data_ptr()), hex(a.spare().data_ptr()), file=sys.stderr)
R.halo_transfer(a)
for _ in range(3):
    R.step(k, a)
torch.cuda.synchronize()
import numpy as np
if os.environ.get("TUNE") == "1":
    print("tune", json.dumps(k.tune(a)), file=sys.stderr)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = int(os.environ.get("N", "10"))
e0.record()
mode = os.environ.get("MODE", "step")
for _ in range(n):
    if mode == "step":
        R.step(k, a)
    elif mode.startswith("mask"):
        R.step(k, a, wrap_mask=int(mode[4:]))
    else:
        R.step(k, a, wrap_mask=0)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
if os.environ.get("ALT") == "1":
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        ev[i][0].record(); R.step(k, a); ev[i][1].record()
    torch.cuda.synchronize()
    t = [x.elapsed_time(y) for x, y in ev]
    print("alt even/odd ms", round(float(np.median(t[0::2])), 4), round(float(np.median(t[1::2])), 4), file=sys.stderr)
import numpy as np
pts = np.prod(shape)
esz = 4 if dt == "float32" else 8
print(json.dumps({"env": {k_: os.environ.get(k_) for k_ in ("LOPE_TILE", "LOPE_ZCHUNK", "LOPE_GRID", "LOPE_FORCE_GENERIC")},
                  "desc": json.loads(k.describe())["tile"] + [json.loads(k.describe()).get("producer_warp")], "ms": round(ms, 4), "gpts": round(pts / ms / 1e6, 1),
                  "GBs": round(2 * esz * pts / ms / 1e6, 1)}), flush=True)
