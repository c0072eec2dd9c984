#!/bin/bash
# Rank-2 y-streaming units, predicated edge stores, DSETP dividend tests: full GPU suite,
# c4/c2/c3 benches (tuned), c4 ncu capture of the tuned plan's kernel.
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/s8_gputest.log 2>&1
for wl in c4 c2 c3 c5 c1; do
  timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu > $O/s8_$wl.jsonl 2> $O/s8_$wl.err
done
timeout 300 python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:1" --steps 20 --warmup 5 --no-e2e --no-cpu \
  --sustained-seconds 1 > $O/s8_c4_yc1.jsonl 2>&1
timeout 300 python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:8" --steps 20 --warmup 5 --no-e2e --no-cpu \
  --sustained-seconds 1 > $O/s8_c4_yc8.jsonl 2>&1
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:^lope_tiled$ --launch-skip 6 -c 1 -o $O/s8_prof_c4_yc8 -f \
  python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:8" --steps 10 --warmup 3 --no-e2e --no-cpu \
  --sustained-seconds 0 > $O/s8_ncu_c4.log 2>&1
ls $O | grep s8_ | head -40
