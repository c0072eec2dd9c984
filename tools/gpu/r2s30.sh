#!/bin/bash
O=gpurun_out
timeout 1200 python tools/machine_bench.py > $O/s30_machine.jsonl 2> $O/s30_machine.err
