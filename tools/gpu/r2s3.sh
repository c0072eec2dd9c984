#!/bin/bash
# Round-2 session 3: full GPU test pass, smoke, default bench, reference arm.
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/s3_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > $O/s3_gputest.log 2>&1
python bench.py > $O/s3_bench_c3.jsonl 2> $O/s3_bench_c3.err
for wl in c4 c5 c1 c2; do
  python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu > $O/s3_$wl.jsonl 2> $O/s3_$wl.err
done
( time python bench.py --impl reference --steps 20 --warmup 5 ) > $O/s3_ref_c3.jsonl 2> $O/s3_ref_c3.err
ls -la $O
