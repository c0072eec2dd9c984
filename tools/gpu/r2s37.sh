#!/bin/bash
O=gpurun_out
for rep in 1 2 3; do python bench.py > $O/s37_c3_$rep.jsonl 2> $O/s37_c3_$rep.err; done
timeout 600 python bench.py --workload c5 --steps 20 --warmup 5 --no-cpu > $O/s37_c5.jsonl 2> $O/s37_c5.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tun or plan" > $O/s37_tests.log 2>&1
