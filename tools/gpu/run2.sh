#!/bin/bash
# Round-2 GPU session 2: new bench contract on c3, the reference arm, ncu traffic of the
# chosen c3 plan, the other workloads, one ncu --set full capture of c4's tiled kernel.
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/r2b2_c3.jsonl 2> $O/r2b2_c3.err
( time python bench.py --impl reference --steps 20 --warmup 5 ) > $O/r2b2_ref_c3.jsonl 2> $O/r2b2_ref_c3.err
python tools/ncu_traffic.py --workload c3 --from-bench $O/r2b2_c3.jsonl > $O/r2b2_traffic_c3.json 2>&1
for wl in c4 c2 c5 c1; do
  python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu > $O/r2b2_$wl.jsonl 2> $O/r2b2_$wl.err
done
PLAN=$(python -c "import sys; sys.path.insert(0,'tools'); import ncu_traffic as t; print(t.plan_arg_from_bench('$O/r2b2_c4.jsonl','c4'))")
echo "c4 plan $PLAN" > $O/r2b2_c4_plan.txt
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:^lope_tiled$ --launch-skip 8 -c 1 -o $O/prof_c4_r2a -f \
  python bench.py --workload c4 --plan "$PLAN" --steps 12 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 \
  > $O/r2b2_ncu_c4.log 2>&1
python tools/ncu_traffic.py --workload c4 --plan "$PLAN" > $O/r2b2_traffic_c4.json 2>&1
ls -la $O
