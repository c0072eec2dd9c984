#!/bin/bash
# ncu capture of c3's in-band z64 plan: round-1 tree vs current tree.
O=gpurun_out
for tree in r1 cur; do
  d=.; [ $tree = r1 ] && d=ab_r1
  extra=""; [ $tree = cur ] && extra="--sustained-seconds 0"
  (cd $d && LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
    --cache-control none -k regex:^lope_tiled$ --launch-skip 8 -c 1 -o /root/repo/$O/s11_prof_c3inb_$tree -f \
    python bench.py --workload c3 --steps 12 --warmup 3 --no-e2e --no-cpu $extra) > $O/s11_ncu_$tree.log 2>&1
done
ls $O | grep s11_
