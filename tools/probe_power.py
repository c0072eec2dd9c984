"""Debug: sustained per-step time, SM clock and board power for one fixed plan."""
import os, sys, pathlib, json, threading, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
if os.environ.get("TUNE") != "1":
    os.environ["LOPE_AUTOTUNE"] = "0"
import torch, numpy as np, pynvml
from paper_1502_03504_b200 import runtime as R, stencils
shape = tuple(int(x) for x in os.environ.get("SHAPE", "1024,1024,1024").split(","))
kir = stencils.by_name(os.environ.get("KERNEL", "lap3d7"))
k = R.CompiledKernel(kir, os.environ.get("DT", "float32"))
fp = kir.footprints[kir.array_params[0]].dims
a = R.HaloArray(shape, [n for n, _ in fp], [p for _, p in fp], os.environ.get("DT", "float32"))
a.fill_hash(1); R.halo_transfer(a)
n = int(os.environ.get("N", "800"))
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []; stop = threading.Event()
def run():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0, pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.01)
tune_rep = k.tune(a) if os.environ.get("TUNE") == "1" else None
for _ in range(3): R.step(k, a)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
t = threading.Thread(target=run, daemon=True); t.start()
for i in range(n):
    ev[i][0].record(); R.step(k, a); ev[i][1].record()
torch.cuda.synchronize(); stop.set(); t.join()
ms = [x.elapsed_time(y) for x, y in ev]
q = n // 8
print(json.dumps({"plan": os.environ.get("LOPE_TILE"), "zc": os.environ.get("LOPE_ZCHUNK"), "pw": os.environ.get("LOPE_PW"),
                  "ms_by_eighth": [round(float(np.median(ms[i*q:(i+1)*q])), 3) for i in range(8)],
                  "sm_mhz": [s[1] for s in samples[::max(1, len(samples)//10)]],
                  "power": [round(s[2]) for s in samples[::max(1, len(samples)//10)]],
                  "capped_frac": round(sum(1 for s in samples if s[3] & 4) / max(1, len(samples)), 2),
                  "tuned": tune_rep["best"] if tune_rep else None,
                  "ms_first_40": [round(x, 2) for x in ms[:40]]}))
