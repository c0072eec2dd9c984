#!/bin/bash
# GPU suite after the describe/candidate changes; config 1 at its default 100 steps; config 4 tuned
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/s60_gputest.log 2>&1
timeout 600 python bench.py --workload c1 > $O/s60_c1.jsonl 2> $O/s60_c1.err
sleep 10
timeout 900 python bench.py --workload c4 > $O/s60_c4.jsonl 2> $O/s60_c4.err
