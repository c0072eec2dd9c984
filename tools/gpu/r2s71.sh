#!/bin/bash
# Final tree: three consecutive driver-style default runs on one box (run-to-run spread)
O=gpurun_out
for rep in 1 2 3; do
  sleep 20
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/s71_bench_c3_$rep.jsonl 2> $O/s71_bench_c3_$rep.err
done
