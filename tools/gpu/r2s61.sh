#!/bin/bash
# Dedicated producer with long z-chunks (deeper ring ahead of the compute warps) on c5 and c3
O=gpurun_out
run() {  # tag workload plan
  sleep 5
  timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s61_$1.jsonl 2> $O/s61_$1.err
}
for rep in 1 2; do
  run c5_inb_$rep c5 1,8,4,8,0,1,0,0:64
  run c5_d12z64_$rep c5 1,16,2,12,1,1,1,0:64
  run c5_d12z32_$rep c5 1,16,2,12,1,1,1,0:32
  run c5_d10z64ns_$rep c5 1,16,2,10,1,1,0,0:64
  run c3_d12z64_$rep c3 1,16,2,12,1,1,1,0:64
  run c3_d12z8_$rep c3 1,16,2,12,1,1,1,0:8
done
