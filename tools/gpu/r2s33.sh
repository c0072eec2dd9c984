#!/bin/bash
O=gpurun_out
timeout 900 python bench.py --workload c5 --steps 20 --warmup 5 --no-cpu > $O/s33_c5.jsonl 2> $O/s33_c5.err
timeout 1500 python tools/fuzz_gpu.py 400 7 > $O/s33_fuzz.log 2>&1
timeout 900 python tools/fuzz_gpu.py 120 8 --decomp > $O/s33_fuzz_decomp.log 2>&1
