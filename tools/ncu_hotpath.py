"""Print, in address order, the SASS lines of an ncu report executed at least N times
(the per-iteration hot path), with their execution counts.
    python tools/ncu_hotpath.py report.ncu-rep N"""
import csv
import subprocess
import sys

rep, n = sys.argv[1], int(float(sys.argv[2]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
h = rows[hi]
ia, isrc, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
cnt = 0
for r in rows[hi + 1:]:
    if len(r) <= ie or not r[ie].strip():
        continue
    try:
        e = int(float(r[ie]))
    except ValueError:
        continue
    if e >= n:
        cnt += 1
        print(f"{r[ia][-5:]} {e:10d}  {r[isrc].strip()[:90]}")
print("lines:", cnt, file=sys.stderr)
