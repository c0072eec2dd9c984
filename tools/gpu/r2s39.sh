#!/bin/bash
# Batched halo-slab copies (lope_copy_boxes): Machine / grid / reference-suite tests, then
# the grid and drop-in Machine throughput again.
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_machine.py tests/test_gpu_reference_suite.py tests/test_gpu_dist.py tests/test_gpu_configs.py -q -x > $O/s39_tests.log 2>&1
timeout 900 python tools/perf_grid.py > $O/s39_grid.jsonl 2> $O/s39_grid.err
timeout 1200 python tools/machine_bench.py > $O/s39_machine.jsonl 2> $O/s39_machine.err
