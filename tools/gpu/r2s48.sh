#!/bin/bash
# fp64 wide-footprint 2-D candidates: GPU suite, tuned config 4 (x2), default bench
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/s48_gputest.log 2>&1
for rep in 1 2; do
  sleep 10
  timeout 600 python bench.py --workload c4 --steps 20 --warmup 5 > $O/s48_c4_$rep.jsonl 2> $O/s48_c4_$rep.err
done
sleep 10
timeout 900 python bench.py > $O/s48_bench_c3.jsonl 2> $O/s48_bench_c3.err
