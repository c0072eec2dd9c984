#!/bin/bash
# Config 4: default plan vs two-warp-wide fp64 tiles, interleaved, 15 s idle before each run
O=gpurun_out
run() {  # tag workload [plan]
  local p=(); [ -n "$3" ] && p=(--plan "$3")
  sleep 15
  timeout 400 python bench.py --workload $2 "${p[@]}" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 4 > $O/s47_$1.jsonl 2> $O/s47_$1.err
}
for rep in 1 2 3; do
  run c4_def_$rep c4 1,16,4,6,1,1,0,0:8
  run c4_w2844d_$rep c4 2,8,4,4,1,1,0,0:8
  run c4_w2845d_$rep c4 2,8,4,5,1,1,0,0:8
  run c4_w2845dy32_$rep c4 2,8,4,5,1,1,0,0:32
done
ls $O | grep s47_ | wc -l
