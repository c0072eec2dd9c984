#!/bin/bash
# c3: two CTAs per SM (two producers and rings per SM) vs the best one-CTA plan.
O=gpurun_out
run() {  # tag plan
  timeout 300 python bench.py --workload c3 --plan "$2" --steps 50 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 2 > $O/s26_$1.jsonl 2> $O/s26_$1.err
}
for rep in 1 2; do
  run best_$rep 1,16,2,12,1,1,1,0:8
  run w16r1_inb_$rep 1,16,1,6,0,2,0,0:64
  run w16r1_ded_$rep 1,16,1,6,1,2,1,0:8
  run w8r2_inb_$rep 1,8,2,6,0,2,0,0:64
  run w8r2_ded_$rep 1,8,2,6,1,2,1,0:8
  run w8r2_ded32_$rep 1,8,2,6,1,2,1,0:32
done
ls $O | grep s26_ | wc -l
