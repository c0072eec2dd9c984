#!/usr/bin/env python
"""DRAM traffic per launch of the dominant kernel under a given execution plan.

    python tools/ncu_traffic.py --workload c3 --from-bench gpurun_out/bench.jsonl
    python tools/ncu_traffic.py --workload c3 --plan 1,16,2,8,1,1,1,0:8
    python tools/ncu_traffic.py --merge gpurun_out/traffic_c3.json ...   # here, afterwards

Runs ``bench.py`` with the plan replayed (``--plan``: no tuning, so the profiled
launches are the plan's) under

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
        --clock-control none --cache-control none -k regex:<kernel> --launch-skip S -c C

and records the median over the captured launches in ``profiles/ncu_traffic.json``
(one entry per workload and plan; ``bench.py`` reports ``roofline.traffic`` only
when its chosen plan has an entry).  ``--cache-control none`` keeps L2 warm between
kernels as in the real loop (ncu's default flush puts the short-z-chunk plans in
their slow mode).  The bench numbers printed under ncu are not bench
values.  GPU box only.
"""

from __future__ import annotations

import argparse
import csv
import json
import pathlib
import statistics
import subprocess
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent
NCU = "/usr/local/cuda/bin/ncu"


def plan_arg_from_bench(path, workload):
    for line in pathlib.Path(path).read_text().splitlines():
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if d.get("config", {}).get("workload") != workload:
            continue
        plans = (d.get("plan") or {}).get("chosen") or {}
        p = next(iter(plans.values()), None)
        if p:
            t = p["tile"]
            cfg = [t[0], t[1], t[2], t[3], p["producer_warp"], 1, p["shfl"], p["nb"]]
            return ",".join(map(str, cfg)) + f":{p['zchunk']}"
    raise SystemExit(f"no {workload} line with a chosen plan in {path}")


def parse_plan(arg):
    cfg, zc, *yb = arg.split(":")
    v = [int(x) for x in cfg.split(",")]
    d = {"tile": v[:4], "producer_warp": v[4], "shfl": v[6], "nb": v[7], "zchunk": int(zc)}
    if yb and int(yb[0]):
        d["yband"] = int(yb[0])
    return d


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--merge":
        # here, after a GPU session: the entries the box printed (its profiles/ is not copied back)
        ents = []
        for f in sys.argv[2:]:
            for line in pathlib.Path(f).read_text().splitlines():
                if line.startswith("{"):
                    e = json.loads(line)
                    if e.get("ncu_kernel_ms", 0) > 1e4:           # entries written before the ns fix
                        e["ncu_kernel_ms"] = round(e["ncu_kernel_ms"] / 1e6, 4)
                    ents.append(e)
        merge(ents)
        print(f"merged {len(ents)} entr{'y' if len(ents) == 1 else 'ies'}")
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True)
    ap.add_argument("--plan")
    ap.add_argument("--from-bench")
    ap.add_argument("--kernel", default="lope_tiled")
    ap.add_argument("--skip", type=int, default=8)
    ap.add_argument("--count", type=int, default=5)
    ap.add_argument("--out", default=str(REPO / "gpurun_out"))
    ap.add_argument("--extra", default="", help="comma-separated further ncu metrics, recorded under 'extra' "
                    "(L2 sectors and hit rates); the entry is then printed only, not merged")
    a = ap.parse_args()
    plan = a.plan or plan_arg_from_bench(a.from_bench, a.workload)
    out = pathlib.Path(a.out)
    out.mkdir(exist_ok=True)
    log = out / f"ncu_traffic_{a.workload}.csv"
    metrics = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum" + (f",{a.extra}" if a.extra else "")
    cmd = [NCU, "--metrics", metrics,
           "--clock-control", "none", "--cache-control", "none", "-k", f"regex:^{a.kernel}$",
           "--launch-skip", str(a.skip), "-c", str(a.count), "--csv", "--log-file", str(log),
           sys.executable, str(REPO / "bench.py"), "--workload", a.workload, "--plan", plan,
           "--steps", str(a.skip + a.count + 2), "--warmup", "3", "--no-e2e", "--no-cpu",
           "--sustained-seconds", "0"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    (out / f"ncu_traffic_{a.workload}.log").write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise SystemExit(f"ncu failed ({res.returncode}); see {out}/ncu_traffic_{a.workload}.log")
    vals = {}
    lines = [l for l in log.read_text().splitlines() if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Kernel Name", "").split("(")[0] != a.kernel:
            continue
        unit = row.get("Metric Unit", "")
        v = float(row["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
                 "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)
        vals.setdefault(row["Metric Name"], []).append(v * scale)
    rd = statistics.median(vals["dram__bytes_read.sum"])
    wr = statistics.median(vals["dram__bytes_write.sum"])
    ms = statistics.median(vals["gpu__time_duration.sum"])
    entry = {"workload": a.workload, "plan": parse_plan(plan), "kernel": a.kernel,
             "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "ncu_kernel_ms": round(ms, 4),
             "launches": len(vals["dram__bytes_read.sum"]),
             "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                       f"--clock-control none --cache-control none, median of {len(vals['dram__bytes_read.sum'])} "
                       f"{a.kernel} launches after {a.skip}, bench.py --workload {a.workload} --plan {plan}"}
    if a.extra:
        entry["extra"] = {m: statistics.median(vals[m]) for m in a.extra.split(",") if m in vals}
    else:
        merge([entry])
    print(json.dumps(entry))


def merge(entries):
    """Add entries to profiles/ncu_traffic.json (replacing the same workload + plan)."""
    p = REPO / "profiles" / "ncu_traffic.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    if "entries" not in d:
        d = {"entries": [], "round1": d}
    for entry in entries:
        d["entries"] = [e for e in d["entries"]
                        if not (e["workload"] == entry["workload"] and e["plan"] == entry["plan"])] + [entry]
    p.write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__":
    main()
