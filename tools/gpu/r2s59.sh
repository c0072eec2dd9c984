#!/bin/bash
# Final-tree evidence: fuzz (new seed), all workloads tuned (c2, c4, c5, c1), default bench + reference arm
O=gpurun_out
timeout 1200 python tools/fuzz_gpu.py 384 20261019 > $O/s59_fuzz.log 2>&1
timeout 900 python tools/fuzz_gpu.py 96 20261020 --decomp > $O/s59_fuzz_decomp.log 2>&1
for w in c2 c4 c5 c1; do
  sleep 10
  timeout 900 python bench.py --workload $w > $O/s59_$w.jsonl 2> $O/s59_$w.err
done
sleep 10
timeout 900 python bench.py > $O/s59_bench_c3.jsonl 2> $O/s59_bench_c3.err
