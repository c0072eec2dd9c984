#!/bin/bash
O=gpurun_out
timeout 900 python tools/perf_grid.py > $O/s38_grid.jsonl 2> $O/s38_grid.err
