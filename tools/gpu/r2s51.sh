#!/bin/bash
# Config 5 DRAM over-read: TMA L2 promotion size and banded unit walks (traffic under ncu,
# then time without it)
O=gpurun_out
X=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct
tr() {  # workload plan promo
  LOPE_L2PROMO=$3 timeout 600 python tools/ncu_traffic.py --workload $1 --plan "$2" --extra $X \
    | sed "s/^{/{\"l2promo\": $3, /" >> $O/s51_traffic.jsonl 2>> $O/s51_traffic.err
}
run() {  # tag workload plan promo
  sleep 5
  LOPE_L2PROMO=$4 timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s51_$1.jsonl 2> $O/s51_$1.err
}
for p in 0 1 3; do tr c5 1,8,4,8,0,1,0,0:64 $p; done
for yb in 2 8; do tr c5 1,8,4,8,0,1,0,0:64:$yb 2; done
tr c5 1,8,4,8,0,1,0,0:32:8 2
tr c3 1,16,2,8,0,1,0,0:64 1
for rep in 1 2; do
  for p in 2 0 1 3; do run c5p${p}_$rep c5 1,8,4,8,0,1,0,0:64 $p; done
  run c5yb8_$rep c5 1,8,4,8,0,1,0,0:64:8 2
  run c5yb2_$rep c5 1,8,4,8,0,1,0,0:64:2 2
  for p in 2 1; do run c3p${p}_$rep c3 1,16,2,8,0,1,0,0:64 $p; done
done
