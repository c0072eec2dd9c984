#!/bin/bash
# Where config 5's extra DRAM reads come from: DRAM and L2 read sectors per tile shape and
# z-chunk (L2 warm between launches, as in the loop)
O=gpurun_out
X=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex_op_write.sum
for spec in "c5 1,16,2,8,0,1,0,1:64" "c5 1,16,2,8,0,1,0,1:128" "c5 1,16,2,8,0,1,0,1:512" "c5 1,16,4,6,0,1,0,0:64" \
            "c5 2,8,2,8,0,1,0,0:64" "c5 1,16,2,12,1,1,1,0:8" "c3 1,16,2,8,0,1,0,0:64" "c3 1,16,2,8,0,1,0,0:256" "c3 1,16,2,12,1,1,1,0:8"; do
  set -- $spec
  timeout 600 python tools/ncu_traffic.py --workload $1 --plan "$2" --extra $X >> $O/s49_traffic.jsonl 2>> $O/s49_traffic.err
done
