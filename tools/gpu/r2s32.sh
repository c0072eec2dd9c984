#!/bin/bash
O=gpurun_out
timeout 900 python bench.py --workload c5 --steps 20 --warmup 5 --no-cpu > $O/s32_c5.jsonl 2> $O/s32_c5.err
timeout 600 python bench.py --workload c1 --steps 100 --warmup 5 --no-cpu > $O/s32_c1.jsonl 2> $O/s32_c1.err
