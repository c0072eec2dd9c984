#!/bin/bash
# Same-box A/B: config 5 default vs 256-column tiles, config 4 default vs 2x8 fp64 tiles.
O=gpurun_out
run() {  # tag workload [plan]
  local p=(); [ -n "$3" ] && p=(--plan "$3")
  timeout 400 python bench.py --workload $2 "${p[@]}" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 4 > $O/s46_$1.jsonl 2> $O/s46_$1.err
}
for rep in 1 2; do
  run c5_nb64_$rep c5 1,16,2,8,0,1,0,1:64
  run c5_w2828_$rep c5 2,8,2,8,0,1,0,0:64
  run c5_w2828z128_$rep c5 2,8,2,8,0,1,0,0:128
  run c4_def_$rep c4 1,16,4,6,1,1,0,0:8
  run c4_w2844_$rep c4 2,8,4,4,0,1,0,0:8
  run c4_w2844d_$rep c4 2,8,4,4,1,1,0,0:8
done
run c5_tuned c5
ls $O | grep s46_ | wc -l
