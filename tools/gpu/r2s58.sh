#!/bin/bash
# DRAM traffic captures for the remaining tuner candidates (roofline.traffic of whichever plan wins)
O=gpurun_out
for spec in "c3 1,16,2,8,0,1,0,1:64" "c3 1,8,4,8,0,1,0,0:64" "c3 1,16,2,8,1,1,1,0:6" "c3 1,16,2,10,1,1,1,0:8" \
            "c3 1,16,2,12,1,1,1,0:6" "c4 1,16,4,6,1,1,0,0:32" "c4 1,16,4,6,0,1,0,0:32" "c4 1,16,4,6,0,1,0,0:1" \
            "c4 2,8,4,6,1,1,0,0:8" "c4 2,8,4,6,1,1,0,0:32" "c2 1,16,2,12,1,1,0,0:1" "c2 1,16,2,12,1,1,0,0:32" \
            "c2 1,16,2,8,1,1,0,0:1" "c2 1,16,2,8,1,1,0,0:32" "c5 1,16,2,8,0,1,0,0:64"; do
  set -- $spec
  timeout 600 python tools/ncu_traffic.py --workload $1 --plan "$2" >> $O/s58_traffic.jsonl 2>> $O/s58_traffic.err
done
