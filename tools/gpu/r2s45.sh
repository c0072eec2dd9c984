#!/bin/bash
# Wide (two-box) tile sweep across configs 2-5, one rep each (runs repeat within 0.3%).
O=gpurun_out
run() {  # tag workload [plan]
  local p=(); [ -n "$3" ] && p=(--plan "$3")
  timeout 400 python bench.py --workload $2 "${p[@]}" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 2 > $O/s45_$1.jsonl 2> $O/s45_$1.err
}
run c3_w2828 c3 2,8,2,8,0,1,0,0:64
run c3_w2828nb c3 2,8,2,8,0,1,0,1:64
run c3_w2828z32 c3 2,8,2,8,0,1,0,0:32
run c3_w28212d c3 2,8,2,12,1,1,1,0:8
run c3_w4428 c3 4,4,2,8,0,1,0,0:64
run c3_w2848 c3 2,8,4,6,0,1,0,0:64
run c5_w2828nb c5 2,8,2,8,0,1,0,1:64
run c5_w2828z32 c5 2,8,2,8,0,1,0,0:32
run c5_w2828z128 c5 2,8,2,8,0,1,0,0:128
run c5_w28212d c5 2,8,2,12,1,1,1,0:8
run c5_w4428 c5 4,4,2,8,0,1,0,0:64
run c5_w2818 c5 2,16,1,8,0,1,0,0:64
run c2_def c2
run c2_w2828 c2 2,8,2,8,1,1,0,0:8
run c2_w4428 c2 4,4,2,8,1,1,0,0:8
run c2_w28212 c2 2,8,2,12,1,1,0,0:8
run c4_def c4
run c4_w2846 c4 2,8,4,4,0,1,0,0:8
run c4_w4446 c4 4,4,4,4,0,1,0,0:8
run c4_w2828 c4 2,8,2,8,0,1,0,0:8
ls $O | grep s45_ | wc -l
