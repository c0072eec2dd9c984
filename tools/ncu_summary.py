"""Summarise an ncu report: key raw metrics, stall reasons, hottest SASS lines."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
d = {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "local_load_bytes", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum"]
for k in keys:
    if k in d:
        print(f"{k:60s} {d[k][0]:8s} {d[k][1]}")
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[1])) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
      and v[1].replace(".", "", 1).isdigit()]
st.sort(key=lambda x: -x[1])
tot = sum(x[1] for x in st) or 1
print("stalls:", ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in st[:8]))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    iw, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [(int(x[iw] or 0), x[ia], x[isrc].strip(), int(x[ie] or 0)) for x in rows[2:] if len(x) > iw]
    n = int(sys.argv[2])
    hot = [x for x in data if x[3] >= n]
    c = collections.Counter()
    for x in hot:
        op = x[2].split()[0] if not x[2].startswith("@") else x[2].split()[1]
        c[op.split(".")[0]] += x[3] / n
    print("instructions per unit-warp (exec >= %d):" % n, round(sum(c.values()), 1))
    print(sorted(((k, round(v, 1)) for k, v in c.items()), key=lambda x: -x[1])[:24])
    for x in sorted(data, key=lambda x: -x[0])[:12]:
        print(x[0], x[1][-5:], x[2][:70], x[3])
