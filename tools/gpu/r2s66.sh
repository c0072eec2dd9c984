#!/bin/bash
# Two CTAs per SM of 8 warps x 4 rows (128 registers each) on c5 / c3
O=gpurun_out
run() {  # tag workload plan
  sleep 5
  timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s66_$1.jsonl 2> $O/s66_$1.err
}
run c5_inb c5 1,8,4,8,0,1,0,0:64
run c5_mb2ns6 c5 1,8,4,6,0,2,0,0:64
run c5_mb2ns5 c5 1,8,4,5,0,2,0,0:64
run c5_mb2ns6nb c5 1,8,4,6,0,2,0,1:64
run c3_mb2ns6 c3 1,8,4,6,0,2,0,0:64
run c3_inb c3 1,16,2,8,0,1,0,0:64
