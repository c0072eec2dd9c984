#!/bin/bash
# Final tree: GPU suite + smoke; ncu --set full of config 4's two-column plan and config 5's in-band plan
O=gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/s64_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/s64_gputest.log 2>&1
NCU="/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --cache-control none -k regex:^lope_tiled$ --launch-skip 8 -c 1"
timeout 900 $NCU -o $O/s64_prof_c4_w2 -f python bench.py --workload c4 --plan 2,8,4,6,1,1,0,0:32 --steps 12 --warmup 3 \
  --no-e2e --no-cpu --sustained-seconds 0 > $O/s64_ncu_c4.log 2>&1
timeout 900 $NCU -o $O/s64_prof_c5_inb -f python bench.py --workload c5 --plan 1,8,4,8,0,1,0,0:64 --steps 12 --warmup 3 \
  --no-e2e --no-cpu --sustained-seconds 0 > $O/s64_ncu_c5.log 2>&1
