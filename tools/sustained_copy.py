"""HBM copy bandwidth burst vs sustained (power-capped) on this B200, as the roofline
denominator for kernels timed inside long runs: torch's device copy of the c3 volume
(4 GiB fp32 read + 4 GiB written, 8.59 GB per copy) back to back for `--seconds`,
CUDA events per copy, NVML clocks/power sampled in a thread.  One JSON line.
    python tools/sustained_copy.py [--seconds 3] [--gib 4]"""
import argparse
import json
import statistics
import threading
import time

import torch


def sampler(stop, out):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        while not stop.is_set():
            out.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            time.sleep(0.01)
    except Exception as e:  # pragma: no cover
        out.append(("error", str(e)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--gib", type=float, default=4.0)
    a = ap.parse_args()
    n = int(a.gib * (1 << 30)) // 4
    x = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
    y = torch.empty_like(x)
    nbytes = 2 * 4 * n
    for _ in range(3):
        y.copy_(x)
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    th = threading.Thread(target=sampler, args=(stop, samples), daemon=True)
    th.start()
    times = []
    t_end = time.time() + a.seconds
    while time.time() < t_end:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        evs[0].record()
        for i in range(20):
            (y.copy_(x) if i % 2 == 0 else x.copy_(y))
            evs[i + 1].record()
        torch.cuda.synchronize()
        times += [evs[i].elapsed_time(evs[i + 1]) for i in range(20)]
    stop.set()
    th.join()
    gbs = [nbytes / (t * 1e-3) / 1e9 for t in times]
    first = gbs[:10]
    last_half = gbs[len(gbs) // 2:]
    ok = [s for s in samples if s[0] != "error"]
    print(json.dumps({
        "what": "torch device copy, 2 x 4 B x n bytes per copy", "bytes_per_copy": nbytes, "copies": len(times),
        "burst_gbs_best": round(max(gbs), 1), "first10_gbs_median": round(statistics.median(first), 1),
        "sustained_gbs_median_last_half": round(statistics.median(last_half), 1),
        "ms_per_copy_median_last_half": round(statistics.median(times[len(times) // 2:]), 4),
        "sm_mhz_median": statistics.median([s[1] for s in ok]) if ok else None,
        "power_w_median": round(statistics.median([s[2] for s in ok]), 1) if ok else None,
        "throttle_reasons_or": hex(int(__import__("functools").reduce(lambda p, q: p | q, [s[3] for s in ok], 0)))
        if ok else None,
    }))


if __name__ == "__main__":
    main()
