#!/bin/bash
# usage: env ... ncu_var.sh label
out=gpurun_out/ncuvar.log
N=8 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control all --clock-control none -k regex:lope_tiled -c 12 --csv --log-file gpurun_out/ncuvar_tmp.csv python tools/probe_perf.py > /dev/null 2>&1
python - "$1" >> $out <<'PY'
import csv, collections, statistics, sys
rows=list(csv.reader(open('gpurun_out/ncuvar_tmp.csv')))
hdr=None; by=collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r and 'Metric Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); by.setdefault(x['ID'],{})[x['Metric Name']]=float(x['Metric Value'])
v=list(by.values())[3:]
print(sys.argv[1], round(statistics.median(d['gpu__time_duration.sum'] for d in v)/1e6,3), round(statistics.median(d['dram__bytes_read.sum'] for d in v)/1e9,2))
PY
