#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_machine.py tests/test_gpu_reference_suite.py -q -x > $O/s41_tests.log 2>&1
timeout 1200 python tools/machine_bench.py > $O/s41_machine.jsonl 2> $O/s41_machine.err
