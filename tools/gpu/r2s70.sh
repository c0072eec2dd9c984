#!/bin/bash
# Former cliffs on the final tree (ragged 1001^3, two-array 3-D, rank 1)
O=gpurun_out
timeout 600 python tools/perf_cliffs.py > $O/s70_cliffs.jsonl 2> $O/s70_cliffs.err
