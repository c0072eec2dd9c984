#!/bin/bash
# c1 temporal blocking: steps per launch / tile height; c3 best plan sustained 5 s.
O=gpurun_out
run() {  # tag env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --workload c1 --steps 100 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 0 > $O/s25_$tag.jsonl 2> $O/s25_$tag.err
}
for rep in 1 2; do
  run tt8_$rep LOPE_AUTOTUNE=0
  run tt16_$rep LOPE_AUTOTUNE=0 LOPE_TBLOCK_TT=16
  run tt4_$rep LOPE_AUTOTUNE=0 LOPE_TBLOCK_TT=4
  run ty12_$rep LOPE_AUTOTUNE=0 LOPE_TBLOCK_TY=12
  run ty56_$rep LOPE_AUTOTUNE=0 LOPE_TBLOCK_TY=56
done
timeout 300 python bench.py --workload c3 --plan "1,16,2,12,1,1,1,0:8" --steps 50 --warmup 5 --no-e2e --no-cpu \
  --sustained-seconds 5 > $O/s25_c3_sust5.jsonl 2> $O/s25_c3_sust5.err
ls $O | grep s25_ | wc -l
