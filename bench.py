#!/usr/bin/env python
"""Benchmark of the LOPe stencil hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl ours|reference]

A *step* is one iteration of ``do it: HALO_TRANSFER(U); do concurrent ... call
K(U)`` over the whole field: one fused liblope_b200.so kernel (launch of step t
plus the periodic halo refresh for step t+1), and at N > 1 the NVLink face
exchange of the partitioned dimension.

Workloads (BASELINE.json configs; default c3, the HBM-roofline headline):
  c1  heat2d   1024^2      fp32  (L2-resident, launch-bound)
  c2  ninept2d 16384^2     fp32
  c3  lap3d7   1024^3      fp32  per GPU (N>1: slab-decomposed along z, weak scaling)
  c4  box5x5   32768^2     fp64  (N>1: the same domain in N slabs along y, strong scaling)
  c5  lap3d7   2048^3      fp32  per GPU

``value`` = interior points x steps (all ranks) / max-over-ranks device time,
in Gpoints/s.  ``e2e`` = the same metric through the public API with the field
in pinned host memory: H2D upload, ``E2E_ITERS`` iterations, D2H download, all
inside the timed region.  ``roofline`` compares the dominant kernel's
algorithmic bytes (2 x sizeof(T) per point update) per launch / its
CUDA-event duration with the measured HBM copy bandwidth.

``--impl reference`` times the reference algorithm on the host CPU (the numpy
port of lopec's vectorised launch in oracle/, all host threads) on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import sys
import threading
import time

REPO = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

WORKLOADS = {
    "c1": dict(kernel="heat2d", shape=(1024, 1024), dtype="float32", split=1, steps=100,
               desc="2D 5-point heat 1024x1024 fp32, halo 1 (config 1: 100 steps)"),
    "c2": dict(kernel="ninept2d", shape=(16384, 16384), dtype="float32", split=1,
               desc="2D 9-point 16384x16384 fp32, halo 1 (config 2)"),
    "c3": dict(kernel="lap3d7", shape=(1024, 1024, 1024), dtype="float32", split=2,
               desc="3D 7-point 1024^3 fp32 per GPU, halo 1 (config 3; N>1 weak-scaled slabs along z)"),
    "c4": dict(kernel="box5x5", shape=(32768, 32768), dtype="float64", split=1, scaling="strong",
               desc="2D 5x5 box 32768x32768 fp64, halo 2 (config 4; N>1: the fixed domain split into "
                    "N slabs along y, 32768 x 32768/N per GPU, strong scaling)"),
    "c5": dict(kernel="lap3d7", shape=(2048, 2048, 2048), dtype="float32", split=2,
               desc="3D 7-point 2048^3 fp32 per GPU, halo 1 (config 5, weak scaling)"),
}
E2E_ITERS = 100
# optional extra untimed warm-up (seconds of load before timing, tuning included); off by
# default: the plan tuner already loads the 3-D configs for ~0.4 s, and on the 2-D ones
# a long warm-up only moves the timed window under the board's power cap
WARM_SECONDS = float(os.environ.get("LOPE_BENCH_WARM_SECONDS", "0"))
SEED = 20260823


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def plan_signature(plan):
    """(tile, producer_warp, shfl, nb, zchunk) of a plan as lope_kernel_describe lists it."""
    if not plan:
        return None
    return (tuple(plan.get("tile", ())), plan.get("producer_warp"), plan.get("shfl"), plan.get("nb"),
            plan.get("zchunk"))


def ncu_traffic(workload, plan):
    """DRAM bytes (read + write) per launch of the dominant kernel, from a committed ncu
    capture of the SAME workload under the SAME execution plan (profiles/ncu_traffic.json,
    written by tools/ncu_traffic.py); None when no capture of this plan exists."""
    p = REPO / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None, "no ncu capture committed"
    try:
        d = json.loads(p.read_text())
    except ValueError:
        return None, "unreadable profiles/ncu_traffic.json"
    sig = plan_signature(plan)
    others = []
    for e in d.get("entries", []):
        if e.get("workload") != workload:
            continue
        if sig is not None and plan_signature(e.get("plan")) == sig:
            return int(e["dram_read_bytes"] + e["dram_write_bytes"]), e.get("source")
        others.append(e.get("plan"))
    return None, f"no capture of this plan (captured plans: {others})"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples = []
        self.power = []
        self.mem_mhz = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:    # pragma: no cover - depends on the box
            log("clock sampling unavailable:", e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.power.append(nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0)
                self.mem_mhz.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_MEM))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join()
        return False

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        p = sorted(self.power)
        mm = sorted(self.mem_mhz)
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(s),
                "power_w_median": round(p[len(p) // 2], 1) if p else None,
                "mem_mhz_median": mm[len(mm) // 2] if mm else None}


# ---------------------------------------------------------------------------
# CPU reference: the reference's own Machine (baseline/_ref lopec) where it can run
# the workload within the time budget, else the threaded numpy port of its
# vectorised launch (oracle/) at full size, else a slab sample of it.

REF_BUDGET_S = float(os.environ.get("LOPE_BENCH_REF_BUDGET_S", "240"))
# single-thread fp64 Machine throughput measured in the survey, used
# only to decide whether K Machine steps fit the budget
MACHINE_GPTS_EST = 0.03


def host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 0


def _lopec():
    """The unmodified reference package, installed under baseline/_ref."""
    ref = REPO / "baseline" / "_ref"
    if (ref / "lopec" / "__init__.py").exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import lopec
    return lopec


def _hash_block(shape, lo, hi, npdt, pool=None, planes_per_task=8):
    """Padded column-major block (the reference's layout, ir.py:189-230) holding the
    device hash field (oracle.hash_planes == lope_fill_hash), zero halo."""
    import numpy as np

    from oracle import lope_oracle as O
    pshape = tuple(m + a + b for m, a, b in zip(shape, lo, hi))
    blk = np.zeros(pshape, dtype=npdt, order="F")
    n = shape[-1]
    inner = tuple(slice(a, a + m) for a, m in zip(lo[:-1], shape[:-1]))

    def fill(z0):
        z1 = min(n, z0 + planes_per_task)
        blk[inner + (slice(lo[-1] + z0, lo[-1] + z1),)] = O.hash_planes(shape, SEED, np.arange(z0, z1), npdt)

    tasks = range(0, n, planes_per_task)
    if pool is not None:
        list(pool.map(fill, tasks))
    else:
        for z in tasks:
            fill(z)
    return blk


def cpu_port(wl, steps, warm, budget_s, shape=None):
    """The threaded numpy port of Machine._halo_exchange + _launch_vector (oracle/),
    all host threads, in the workload's dtype.  Full size when the time budget and
    host memory allow, otherwise a slab of the slowest axis (stated in `sample`)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import lope_oracle as O
    from paper_1502_03504_b200 import stencils

    kir = stencils.by_name(wl["kernel"])
    npdt = np.float32 if wl["dtype"] == "float32" else np.float64
    shape = list(shape or wl["shape"])
    full = list(shape)
    fp = kir.footprints[kir.array_params[0]].dims
    lo, hi = [n for n, _ in fp], [p for _, p in fp]
    esz = np.dtype(npdt).itemsize
    pts = int(np.prod(shape))
    threads = os.cpu_count() or 1
    pool = ThreadPoolExecutor(threads)
    # calibrate on a slab of ~16M points, then fit the budget and half the host memory
    # (block + snapshot)
    inner = pts // shape[-1]
    probe = list(shape)
    probe[-1] = max(4, min(shape[-1], (1 << 24) // max(1, inner)))
    pblk = _hash_block(probe, lo, hi, npdt, pool)
    t0 = time.perf_counter()
    O.threaded_machine_step(pblk, lo, hi, kir, None, npdt, pool, threads)
    rate = int(np.prod(probe)) / max(1e-9, time.perf_counter() - t0)
    del pblk
    frac = min(1.0, budget_s / max(1e-9, (steps + warm) * pts / rate))
    ram = host_ram_bytes()
    if ram:
        frac = min(frac, 0.5 * ram / (2.2 * pts * esz))
    if frac < 1.0:
        shape[-1] = max(4, int(shape[-1] * frac))
    t_gen = time.perf_counter()
    blk = _hash_block(shape, lo, hi, npdt, pool)
    t_gen = time.perf_counter() - t_gen
    for _ in range(warm):
        O.threaded_machine_step(blk, lo, hi, kir, None, npdt, pool, threads)
    per = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.threaded_machine_step(blk, lo, hi, kir, None, npdt, pool, threads)
        per.append(time.perf_counter() - t0)
    pool.shutdown()
    el = sum(per)
    pts = int(np.prod(shape))
    same = shape == full
    return {"value": pts * steps / el / 1e9 if el > 0 else None, "unit": "Gpoints/s", "cores": threads,
            "kind": "port", "same_config": same, "steps": steps, "seconds": round(el, 3),
            "ms_per_step": round(1e3 * el / max(1, steps), 3),
            "sample": (f"{steps} step(s) of {kir.name} on {'x'.join(map(str, shape))} {wl['dtype']}"
                       f"{' (the full workload)' if same else ' (slab of the full ' + 'x'.join(map(str, full)) + ')'}"
                       f": numpy port of lopec Machine._halo_exchange + _launch_vector (oracle/lope_oracle.py "
                       f"threaded_machine_step), {threads} host threads, {el:.1f} s timed, input generation "
                       f"{t_gen:.1f} s untimed")}


def reference_machine(wl, steps, warm):
    """The reference's own ``Machine`` (baseline/_ref, unmodified) running the config's
    program -- HALO_TRANSFER + device launch per iteration (runtime.py:308-337) -- in
    fp64, its only precision, on one host thread (numpy ufuncs are single-threaded)."""
    import numpy as np

    from oracle.lope_programs import program_text
    lopec = _lopec()
    from lopec.runtime import Machine, RunConfig
    prog, diags = lopec.parse_source(program_text(wl["kernel"]), f"{wl['kernel']}.lope")
    if prog is None or diags:
        raise RuntimeError(f"reference frontend rejected the program: {diags}")
    chk = lopec.check_program(prog)
    shape = tuple(wl["shape"])
    field = np.asfortranarray(_hash_block(shape, [0] * len(shape), [0] * len(shape), np.float64))
    if warm:
        Machine(chk, RunConfig(images=1, steps=warm), field.copy()).run()
    m = Machine(chk, RunConfig(images=1, steps=steps), field)
    t0 = time.perf_counter()
    m.run()
    el = time.perf_counter() - t0
    pts = int(np.prod(shape))
    return {"value": pts * steps / el / 1e9, "unit": "Gpoints/s", "cores": 1, "kind": "reference",
            "same_config": True, "steps": steps, "seconds": round(el, 3),
            "ms_per_step": round(1e3 * el / max(1, steps), 3), "precision": "f64",
            "sample": (f"lopec.Machine(check, RunConfig(images=1, steps={steps})).run() from baseline/_ref "
                       f"(unmodified reference) on {wl['kernel']} {'x'.join(map(str, shape))}, fp64 (the "
                       f"reference's only precision), 1 numpy thread of {os.cpu_count()} host cores, "
                       f"{el:.2f} s")}


def cpu_reference_full(wl, steps, warm, budget_s=REF_BUDGET_S):
    """The reference arm's measurement: the reference Machine when the config is rank <= 2
    and K + W of its steps fit the budget, else the port (full size when it fits)."""
    import numpy as np
    pts = int(np.prod(wl["shape"]))
    if len(wl["shape"]) <= 2 and (steps + warm) * pts / (MACHINE_GPTS_EST * 1e9) <= budget_s:
        try:
            return reference_machine(wl, steps, warm)
        except Exception as e:             # pragma: no cover - reference install missing
            log("reference Machine unavailable, timing the port:", e)
    return cpu_port(wl, steps, warm, budget_s)


def run_reference_arm(args, wl):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    res = cpu_reference_full(wl, steps, warm)
    line = {
        "metric": "stencil Gpoints/s & HBM GB/s (% of 8 TB/s roofline) at 1/2/4/8 B200 vs CPU ref",
        "impl": "reference", "value": res["value"], "unit": "Gpoints/s", "n_gpus": ws,
        "steps": steps, "warmup": warm,
        # measured per step of what ran (the full workload unless `same_config` is false)
        "ms_per_step": res["ms_per_step"],
        "higher_is_better": True,
        "scaling": wl.get("scaling", "weak"), "vs_baseline": None,
        "dtype": "f64" if res.get("precision") == "f64" or wl["dtype"] == "float64" else "f32",
        "data": "synthetic (splitmix64 U(-1,1) hash field, the GPU arm's input)",
        "config": {"workload": args.workload, "desc": wl["desc"], "kernel": wl["kernel"],
                   "shape_per_gpu": list(wl["shape"]), "same_config": bool(res.get("same_config"))},
        "cpu_baseline": res,
        "e2e": {"value": res["value"], "unit": "Gpoints/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


def run_gpu_arm(args, wl):
    import numpy as np
    import torch

    from paper_1502_03504_b200 import _lib, stencils
    from paper_1502_03504_b200 import runtime as R

    ws, rank, local = dist_env()
    # one process per GPU; LOPE_BENCH_BACKEND=gloo lets a one-GPU box run the N>1 code
    # path with all ranks sharing the device (a functional check, not a measurement)
    backend = os.environ.get("LOPE_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    kir = stencils.by_name(wl["kernel"])
    kern = R.CompiledKernel(kir, wl["dtype"])
    exchange_kind = None
    fp = kir.footprints[kir.array_params[0]].dims
    lo, hi = [n for n, _ in fp], [p for _, p in fp]
    strong = wl.get("scaling", "weak") == "strong"
    gshape = tuple(wl["shape"]) if strong else tuple(wl["shape"][:-1]) + (wl["shape"][-1] * ws,)
    if gshape[-1] % ws:
        raise SystemExit(f"{args.workload}: {gshape[-1]} planes do not split over {ws} GPUs")
    shape = tuple(gshape[:-1]) + (gshape[-1] // ws,)      # this rank's slab
    esz = 4 if wl["dtype"] == "float32" else 8
    points = int(np.prod(shape))
    stream = torch.cuda.current_stream()

    if ws > 1:
        from paper_1502_03504_b200 import dist as D
        field = D.SlabArray(shape, lo, hi, wl["dtype"], group=group)
        gorg = [0] * (len(shape) - 1) + [shape[-1] * rank]
        field.block.fill_hash(SEED, list(gshape), gorg)
        # fused exchange: the kernel stores boundary planes into the neighbours' halos
        # through CUDA IPC peer memory; NCCL send/recv overlapped with the interior if
        # the peer mapping is unavailable
        exchange_kind = "fused-peer-store"
        try:
            if os.environ.get("LOPE_EXCHANGE", "peer") != "peer":
                raise RuntimeError("LOPE_EXCHANGE selects NCCL")
            stepper = D.PeerSlabStepper(kern, field, group=group)
        except Exception as e:             # pragma: no cover - depends on the node
            log("peer exchange unavailable, using NCCL send/recv:", e)
            exchange_kind = "nccl-send-recv-overlapped (lope_halo_exchange)"
            stepper = D.SlabStepper(kern, field, native=backend == "nccl", group=group)
        stepper.exchange()

        def do_step():
            stepper.step()
        arr = field.block
    else:
        arr = R.HaloArray(shape, lo, hi, wl["dtype"])
        arr.fill_hash(SEED)
        R.halo_transfer(arr)

        def do_step():
            R.step(kern, arr)

    if args.plan:
        # replay a recorded plan instead of tuning (profiling captures of one plan)
        import ctypes
        os.environ["LOPE_AUTOTUNE"] = "0"
        cfg, zc, *yb = args.plan.split(":")
        vals = [int(v) for v in cfg.split(",")]
        _lib.check(_lib.lib().lope_plan_set_variant(kern.handle, ctypes.byref(arr.layout), (1 << arr.rank) - 1,
                                                    (ctypes.c_int32 * 8)(*vals), int(zc), int(yb[0]) if yb else 0,
                                                    None),
                   "lope_plan_set_variant")
    # plan selection (runtime.PlanTuner): real steps under each candidate plan, part
    # of setup like compilation; the timed steps run the chosen plan
    tune_steps = 0
    t_tune = time.perf_counter()
    if ws > 1:
        tune_steps = stepper.tune()
    else:
        while kern.tuning(arr, (1 << arr.rank) - 1):
            do_step()
            tune_steps += 1
    torch.cuda.synchronize()
    tune_secs = time.perf_counter() - t_tune
    t_w = time.perf_counter()
    for _ in range(args.warmup):
        do_step()
    torch.cuda.synchronize()
    warm_secs = time.perf_counter() - t_w
    # optional: extra untimed steps until the warm-up (tuning included) has lasted
    # WARM_SECONDS -- a step count every rank agrees on, since the multi-GPU steps
    # synchronise
    step_est = warm_secs / max(1, args.warmup)
    extra = int(math.ceil(max(0.0, WARM_SECONDS - tune_secs - warm_secs) / max(step_est, 1e-6)))
    extra = min(extra, 10000)
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([extra], device=dev, dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        extra = int(t.item())
    for _ in range(extra):
        do_step()
    torch.cuda.synchronize()
    graph = None
    if ws == 1 and points * esz < 64 << 20:
        # L2-resident field (config 1): launch-bound, so the K timed steps are captured
        # once as a CUDA graph (after the plain warm-up steps) and replayed once
        graph = R.StepGraph(kern, arr, args.steps)
        graph.replay()                 # first replay uploads the graph: keep it untimed
        torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # timed region: exactly K steps, per-step events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_all0, t_all1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    barrier()
    with ClockSampler(local) as clk:
        t_all0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                ev[i][0].record(stream)
                do_step()
                ev[i][1].record(stream)
        t_all1.record(stream)
        torch.cuda.synchronize()
    steps_done = graph.steps if graph is not None else args.steps
    barrier()
    launches = _lib.launch_count() - l0
    total_ms = t_all0.elapsed_time(t_all1)
    if graph is not None:
        launches = graph.launches      # one graph replay: the host counter saw the captures
        per_step = [total_ms / steps_done]
    else:
        per_step = [a.elapsed_time(b) for a, b in ev]
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / steps_done
    value = points * ws * steps_done / (total_ms / 1e3) / 1e9

    # dominant kernel: the fused step kernel, one launch per step (N > 1: the step's
    # device time on this rank includes the stream wait on the neighbours' flags, so
    # the fraction is a lower bound for the kernel)
    kernel_ms = sorted(per_step)[len(per_step) // 2]
    alg_bytes = 2 * esz * points
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    chosen = json.loads(kern.describe()).get("plans") or {}
    plan = next(iter(chosen.values()), None)
    if graph is not None:
        plan = {"kernel": "lope_tblock"}
    if ws == 1:
        traffic, traffic_src = ncu_traffic(args.workload, plan)
    else:       # the captures are of the one-GPU workload; a slab's geometry differs
        traffic, traffic_src = None, "no capture of the N>1 slab geometry"
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": peak_src, "alg_bytes_per_launch": alg_bytes,
                "kernel_ms": round(kernel_ms, 4),
                "step_ms_min_med_max": [round(min(per_step), 4), round(sorted(per_step)[len(per_step) // 2], 4),
                                        round(max(per_step), 4)],
                "pct_of_8TBs": round(100 * alg_bytes / (kernel_ms / 1e3) / 8e12, 1)}

    # sustained: the same step for >= `--sustained-seconds` of device time right after
    # the timed window (the board's power cap engages within ~0.5 s on every large
    # config; this is the rate a long run settles at)
    sustained = None
    if args.sustained_seconds > 0:
        per_launch = ms_per_step * (steps_done if graph is not None else 1)
        nrep = int(min(50000, max(3, math.ceil(1e3 * args.sustained_seconds / max(per_launch, 1e-4)))))
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nrep)]
        barrier()
        with ClockSampler(local) as sclk:
            for i in range(nrep):
                sev[i][0].record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    do_step()
                sev[i][1].record(stream)
            torch.cuda.synchronize()
        barrier()
        d = sorted(a.elapsed_time(b) / (steps_done if graph is not None else 1) for a, b in sev)
        med = d[len(d) // 2]
        tot = sum(d) * (steps_done if graph is not None else 1) / 1e3
        sustained = {"steps": nrep * (steps_done if graph is not None else 1), "seconds": round(tot, 3),
                     "ms_per_step_median": round(med, 4),
                     "value_median": round(points * ws / (med / 1e3) / 1e9, 3),
                     "pct_of_8TBs_median": round(100 * 2 * esz * points / (med / 1e3) / 8e12, 1),
                     "frac_of_measured_peak_median": round(2 * esz * points / (med / 1e3) / 1e9 / measured_peak()[0], 4),
                     "clocks": sclk.summary(),
                     "note": "per-rank device time of rank 0" if ws > 1 else "device time, CUDA events per step"}
        pw = (sustained["clocks"] or {}).get("power_w_median")
        if pw:
            # board energy per billion point updates at the capped steady state
            sustained["joules_per_gpoint"] = round(pw / (points / (med / 1e3) / 1e9), 4)

    # the device-timed blocks are done: free them before the e2e batch allocates its
    # own (config 5: 69 GB per ping-pong pair; with them alive only one batch slot fits)
    used_graph = graph is not None
    do_step = arr = graph = field = stepper = None
    torch.cuda.empty_cache()

    # e2e through the public API, host buffers, H2D + E2E_ITERS iterations + D2H timed
    e2e = None
    if not args.no_e2e:
        e2e = e2e_measure(args, wl, kern, lo, hi, shape, gshape, esz, group, ws, rank, dev)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        # bounded: a couple of full-size steps (config 1: the reference Machine itself)
        small = int(np.prod(wl["shape"])) <= (1 << 22)
        cpu = cpu_reference_full(wl, steps=args.steps if small else 2, warm=1 if small else 0,
                                 budget_s=args.cpu_seconds)

    del arr
    if rank == 0:
        line = {
            "metric": "stencil Gpoints/s & HBM GB/s (% of 8 TB/s roofline) at 1/2/4/8 B200 vs CPU ref",
            "value": round(value, 3), "unit": "Gpoints/s", "n_gpus": ws, "steps": args.steps,
            "cuda_graph": used_graph,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": wl.get("scaling", "weak"), "vs_baseline": None,
            "dtype": "f32" if wl["dtype"] == "float32" else "f64",
            "data": "synthetic (splitmix64 U(-1,1) field generated on device)",
            "config": {"workload": args.workload, "desc": wl["desc"], "kernel": wl["kernel"],
                       "shape_per_gpu": list(shape), "global_shape": list(gshape),
                       "halo": [lo, hi], "parallelism": f"slab{ws}" if ws > 1 else "single",
                       "exchange": exchange_kind if ws > 1 else "in-kernel periodic images",
                       "l2": "inputs larger than L2 (no flush needed)" if alg_bytes > 4 * 126e6
                             else "L2-resident working set (config 1); HBM fraction informational",
                       "hbm_gbs_alg": round(alg_bytes * ws / (ms_per_step / 1e3) / 1e9 / ws, 1)},
            "plan": {"chosen": json.loads(kern.describe()).get("plans"), "timed_window": chosen,
                     "tuning_steps": tune_steps,
                     "extra_warmup_steps": extra,
                     "watchdog_fallback": [t.report.get("fallback") for t in kern._tuners.values()]},
            "roofline": roofline,
            "sustained": sustained,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def e2e_measure(args, wl, kern, lo, hi, shape, gshape, esz, group, ws, rank, dev):
    """Public API, host (pinned) buffers: upload, E2E_ITERS iterations, download.

    The input is this rank's slab of the hash field (the device-timed run's input, so
    data-dependent paths such as flagged divisions see the same values), produced on
    the device and downloaded into the pinned buffer before the timed region."""
    import numpy as np
    import torch

    from paper_1502_03504_b200 import runtime as R

    nbytes = int(np.prod(shape)) * esz
    tdt = torch.float32 if esz == 4 else torch.float64
    host_in = torch.empty(nbytes // esz, dtype=tdt, pin_memory=True)
    src = R.HaloArray(shape, lo, hi, wl["dtype"])
    src.fill_hash(SEED, list(gshape), [0] * (len(shape) - 1) + [shape[-1] * rank])
    src.download(host_in.data_ptr())
    torch.cuda.synchronize()
    del src
    torch.cuda.empty_cache()
    host_out = torch.empty_like(host_in, pin_memory=True)
    if ws > 1:
        from paper_1502_03504_b200 import dist as D

        def call():
            D.run_pinned(kern, shape, lo, hi, wl["dtype"], host_in, host_out, E2E_ITERS, group)
    else:
        def call():
            R.run_pinned(kern, shape, lo, hi, wl["dtype"], host_in, host_out, E2E_ITERS)
    call()                              # warm-up (allocation, module load)
    torch.cuda.synchronize()
    reps = 2
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    pts = int(np.prod(shape)) * ws * E2E_ITERS * reps
    single = {"value": round(pts / el / 1e9, 3), "unit": "Gpoints/s",
              "h2d_bytes_per_step": nbytes // E2E_ITERS, "d2h_bytes_per_step": nbytes // E2E_ITERS,
              "iters_per_call": E2E_ITERS, "calls": reps, "seconds": round(el, 4),
              "api": "runtime.run_pinned (HaloArray upload, iterate, gather)",
              "input": "hash field slab in pinned host memory (column-major)"}
    if ws > 1 or args.e2e_fields <= 1 or nbytes < (256 << 20):
        # small fields (config 1: 4 MB) are bound by per-call host work, which a batch
        # of streams and events only adds to: single calls are the end-to-end number
        return single
    # a batch of independent fields through runtime.run_pinned_batch: field i+1 uploads
    # and field i-1 downloads while field i iterates (3 device slots, 3 streams)
    nf = args.e2e_fields
    if nbytes > (16 << 30):
        nf = min(nf, 4)                 # 34 GB fields (config 5): keep the run short
    R.run_pinned_batch(kern, shape, lo, hi, wl["dtype"], [host_in] * 2, [host_out] * 2, 2)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R.run_pinned_batch(kern, shape, lo, hi, wl["dtype"], [host_in] * nf, [host_out] * nf, E2E_ITERS)
    torch.cuda.synchronize()
    elb = time.perf_counter() - t0
    ptsb = int(np.prod(shape)) * E2E_ITERS * nf
    return {"value": round(ptsb / elb / 1e9, 3), "unit": "Gpoints/s",
            "h2d_bytes_per_step": nbytes // E2E_ITERS, "d2h_bytes_per_step": nbytes // E2E_ITERS,
            "iters_per_field": E2E_ITERS, "fields": nf, "seconds": round(elb, 4),
            "api": "runtime.run_pinned_batch (3 device slots on 3 streams: the H2D of field i+1 "
                   "and the D2H of field i-1 overlap the iterations of field i)",
            "input": "hash field slab in pinned host memory (column-major), one upload and one "
                     "download per field, all inside the timed region",
            "single_call": single}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the configuration's own step count, config 1: 100; else 50)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-fields", type=int, default=32,
                    help="independent fields in the pipelined e2e batch (1: single calls only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--sustained-seconds", type=float, default=1.0)
    ap.add_argument("--plan", default=None,
                    help="replay a plan 'bxw,wy,ry,ns,pw,mb,sh,nb:zchunk[:yband]' instead of tuning (ncu captures)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    wl = WORKLOADS[args.workload]
    if args.steps is None:
        args.steps = wl.get("steps", 50)
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != ws_env:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws_env}; launch N>1 with torchrun "
            f"(--nproc-per-node N); reporting n_gpus={ws_env}")
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_gpu_arm(args, wl)


if __name__ == "__main__":
    main()
