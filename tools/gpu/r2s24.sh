#!/bin/bash
# Multi-array kernel: plain-store fast path, pairs on/off; its parity tests.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py tests/test_gpu_parity.py -q -x -k "multi" > $O/s24_tests.log 2>&1
for rep in 1 2; do
  timeout 300 python tools/perf_cliffs.py --cases two3d > $O/s24_two3d_pair_$rep.jsonl 2>&1
  LOPE_NVRTC_DEFS=-DLOPE_NO_PAIR timeout 300 python tools/perf_cliffs.py --cases two3d > $O/s24_two3d_np_$rep.jsonl 2>&1
done
ls $O | grep s24_
