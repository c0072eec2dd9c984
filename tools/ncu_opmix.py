"""Dynamic opcode mix of one kernel in an ncu report (source page, SASS view): executed
warp-instructions per opcode, per point when `points` is given.
    python tools/ncu_opmix.py report.ncu-rep [points]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
pts = float(sys.argv[2]) if len(sys.argv) > 2 else None
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
h = rows[hi]
isrc, ie = h.index("Source"), h.index("Instructions Executed")
iw = h.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in h else None
ops, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= ie or not r[ie].strip():
        continue
    try:
        n = int(float(r[ie]))
    except ValueError:
        continue
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    ops[op] += n
    tot += n
    if iw is not None and r[iw].strip():
        stall[op] += int(float(r[iw]))
print(f"total warp-instructions {tot:.4g}" + (f"  = {32 * tot / pts:.2f} thread-instructions per point" if pts else ""))
st = sum(stall.values()) or 1
for op, n in ops.most_common(28):
    per = f" {32 * n / pts:6.2f}/pt" if pts else ""
    print(f"  {op:12s} {n:14d} {100 * n / tot:5.1f}%{per}  stall-samples {100 * stall[op] / st:5.1f}%")
