#!/bin/bash
# Round-2 measurement set: smoke, GPU suite, every workload (tuned), the reference arm
# (c3), cliffs, one ncu --set full capture of c3's best plan.
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/s19_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/s19_gputest.log 2>&1
python bench.py > $O/s19_bench_c3.jsonl 2> $O/s19_bench_c3.err
for wl in c2 c4 c5 c1; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 > $O/s19_$wl.jsonl 2> $O/s19_$wl.err
done
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > $O/s19_ref_c3.jsonl 2> $O/s19_ref_c3.err
( time timeout 900 python bench.py --impl reference --workload c1 --steps 20 --warmup 5 ) > $O/s19_ref_c1.jsonl 2> $O/s19_ref_c1.err
timeout 300 python tools/perf_cliffs.py > $O/s19_cliffs.jsonl 2>&1
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:^lope_tiled$ --launch-skip 8 -c 1 -o $O/s19_prof_c3_best -f \
  python bench.py --workload c3 --plan "1,16,2,12,1,1,1,0:8" --steps 12 --warmup 3 --no-e2e --no-cpu \
  --sustained-seconds 0 > $O/s19_ncu_c3.log 2>&1
ls $O | grep s19_
