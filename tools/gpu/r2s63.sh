#!/bin/bash
# Temporal blocking: 16-byte stores of image-free vectors in the last step (A/B on config 1)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal or graph or config1 or c1" > $O/s63_tests.log 2>&1
for rep in 1 2 3; do
  for v in vec scalar; do
    D=""; [ $v = scalar ] && D="-DLOPE_TB_SCALAR_STORE"
    LOPE_NVRTC_DEFS="$D" timeout 300 python bench.py --workload c1 --no-e2e --no-cpu > $O/s63_c1_${v}_$rep.jsonl 2> $O/s63_c1_${v}_$rep.err
  done
done
