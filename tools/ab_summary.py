#!/usr/bin/env python
"""Summarise tools/gpu/ab.sh results: per spec, bench ms/step (window, sustained) and
the ncu counters of the lope_tiled launches (median)."""
import csv
import json
import pathlib
import statistics
import sys

O = pathlib.Path("gpurun_out")
tag = sys.argv[1]
for line in (O / f"ab_{tag}_index.txt").read_text().splitlines():
    i, wl, plan, *defs = line.split()
    b = json.loads((O / f"ab_{tag}_{i}.jsonl").read_text().splitlines()[-1])
    vals = {}
    rows = [r for r in (O / f"ab_{tag}_{i}.csv").read_text().splitlines() if r.startswith('"')]
    for r in csv.DictReader(rows):
        vals.setdefault(r["Metric Name"], []).append(float(r["Metric Value"].replace(",", "")))
    med = {k: statistics.median(v) for k, v in vals.items()}
    pts = 1
    for m in b["config"]["shape_per_gpu"]:
        pts *= m
    print(f"{i} {wl} {plan} {' '.join(defs)}")
    print(f"   bench {b['ms_per_step']:.4f} ms  sustained {b['sustained']['ms_per_step_median']:.4f} ms "
          f"({b['sustained']['pct_of_8TBs_median']}% of 8TB/s, sm {b['sustained']['clocks']['sm_mhz']} MHz, "
          f"{b['sustained']['clocks'].get('power_w_median')} W)")
    print(f"   ncu {med['gpu__time_duration.sum'] / 1e6:.4f} ms  inst/pt {32 * med['smsp__inst_executed.sum'] / pts:.2f}  "
          f"dram {(med['dram__bytes_read.sum'] + med['dram__bytes_write.sum']) / 1e9:.3f} GB  "
          f"issue {med['smsp__issue_active.avg.pct_of_peak_sustained_active']:.1f}%  "
          f"fp64 {med['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:.1f}%  "
          f"alu {med['sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active']:.1f}%  "
          f"lsu {med['sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']:.1f}%")
