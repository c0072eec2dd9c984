#!/bin/bash
# Shorter tuning: default bench x3, c5, and the tuner-related GPU tests.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -k "tun or c5 or ragged" > $O/s31_tests.log 2>&1
for rep in 1 2 3; do
  python bench.py > $O/s31_c3_$rep.jsonl 2> $O/s31_c3_$rep.err
done
timeout 600 python bench.py --workload c5 --steps 20 --warmup 5 --no-cpu > $O/s31_c5.jsonl 2> $O/s31_c5.err
ls $O | grep s31_
