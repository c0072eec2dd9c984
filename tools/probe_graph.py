"""Debug: config-1 style CUDA-graph timing for small fields under tile-config overrides."""
import os, sys, pathlib, json
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_1502_03504_b200 import runtime as R, stencils
shape = tuple(int(x) for x in os.environ.get("SHAPE", "1024,1024").split(","))
kir = stencils.by_name(os.environ.get("KERNEL", "heat2d"))
k = R.CompiledKernel(kir, "float32")
a = R.HaloArray(shape, [1, 1], [1, 1], "float32")
a.fill_hash(1)
R.halo_transfer(a)
n = 100
if os.environ.get("MULTI") == "1":
    class _G:
        steps = n
        def __init__(self):
            torch.cuda.synchronize()
            s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                R.multi_step(k, a, n)
            torch.cuda.current_stream().wait_stream(s)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                R.multi_step(k, a, n)
        def replay(self):
            self.graph.replay()
    g = _G()
else:
    g = R.StepGraph(k, a, n)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / n
print(json.dumps({"env": os.environ.get("LOPE_TILE"), "mb": os.environ.get("LOPE_MB"), "desc": json.loads(k.describe())["tile"],
                  "us_per_step": round(us, 2), "gpts": round(shape[0] * shape[1] / us / 1e3, 1)}), flush=True)
