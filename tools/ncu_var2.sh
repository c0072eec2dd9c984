#!/bin/bash
N=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:lope_tiled -c 6 --csv --log-file gpurun_out/ncuv2_tmp.csv python tools/probe_perf.py > /dev/null 2>&1
python - "$1" >> gpurun_out/ncuv2.log <<'PY'
import csv, collections, statistics, sys
rows=list(csv.reader(open('gpurun_out/ncuv2_tmp.csv')))
hdr=None; by=collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r and 'Metric Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); by.setdefault(x['ID'],{})[x['Metric Name']]=float(x['Metric Value'])
v=list(by.values())[3:]
print(sys.argv[1], round(statistics.median(d['gpu__time_duration.sum'] for d in v)/1e6,3), 'ms', round(statistics.median(d['dram__bytes_read.sum'] for d in v)/1e9,2), 'GB rd', round(statistics.median(d['dram__bytes_write.sum'] for d in v)/1e9,2), 'GB wr', round(statistics.median(d['lts__t_sector_hit_rate.pct'] for d in v),1), '% L2 hit')
PY
