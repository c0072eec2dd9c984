#!/bin/bash
# Launch list of the final default bench (kernel share of the step), as the contract asks
O=gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/s68_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 \
  > $O/s68_launches_c3.log 2>&1
