#!/bin/bash
# Temporal blocking: task index division in fp32 (corrected) vs integer division (A/B on config 1)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal or graph or config1 or c1" > $O/s69_tests.log 2>&1
for rep in 1 2 3; do
  for v in fdiv idiv; do
    D=""; [ $v = idiv ] && D="-DLOPE_TB_INTDIV"
    LOPE_NVRTC_DEFS="$D" timeout 300 python bench.py --workload c1 --no-e2e --no-cpu > $O/s69_c1_${v}_$rep.jsonl 2> $O/s69_c1_${v}_$rep.err
  done
done
