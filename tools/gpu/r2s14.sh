#!/bin/bash
# ncu of c3 in-band z64 for the current tree without pairs and with the round-1 store code.
O=gpurun_out
LOPE_NVRTC_DEFS="-DLOPE_NO_PAIR -DLOPE_OLD_STORE" LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 /usr/local/cuda/bin/ncu --set full \
  --import-source on --clock-control none --cache-control none -k regex:^lope_tiled$ --launch-skip 8 -c 1 \
  -o $O/s14_prof_c3inb_npos -f python bench.py --workload c3 --steps 12 --warmup 3 --no-e2e --no-cpu \
  --sustained-seconds 0 > $O/s14_ncu.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "batch or pinned" > $O/s14_tests.log 2>&1
python bench.py --workload c3 --steps 20 --warmup 5 --no-cpu > $O/s14_c3.jsonl 2> $O/s14_c3.err
ls $O | grep s14_
