#!/bin/bash
# c3: 32 warps x 1 row per lane (twice the warps, 64 registers) vs the current best plan.
O=gpurun_out
run() {  # tag plan
  timeout 300 python bench.py --workload c3 --plan "$2" --steps 50 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 2 > $O/s23_$1.jsonl 2> $O/s23_$1.err
}
for rep in 1 2; do
  run best_$rep 1,16,2,12,1,1,1,0:8
  run w32_z64_$rep 1,32,1,8,0,1,0,0:64
  run w32_z16_$rep 1,32,1,8,0,1,0,0:16
  run w32s_z64_$rep 1,32,1,8,0,1,1,0:64
  run w32_n12_z64_$rep 1,32,1,12,0,1,0,0:64
  run w24_z64_$rep 1,24,1,8,0,1,0,0:64
done
ls $O | grep s23_ | wc -l
