#!/bin/bash
# c4 regression: one ncu --set full capture of box5x5's lope_tiled in the old tree and now.
O=gpurun_out
for v in old cur; do
  d=.; [ $v = old ] && d=ab_old
  (cd $d && /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --cache-control none \
    -k regex:^lope_tiled$ --launch-skip 6 -c 1 -o /root/repo/$O/s7_prof_c4_$v -f \
    python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:1" --steps 10 --warmup 3 --no-e2e --no-cpu \
    --sustained-seconds 0) > $O/s7_ncu_c4_$v.log 2>&1
done
(cd . && timeout 300 python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:1" --steps 20 --warmup 5 --no-e2e --no-cpu \
  --sustained-seconds 1) > $O/s7_c4_cur.jsonl 2>&1
ls $O | grep s7
