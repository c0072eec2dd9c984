#!/bin/bash
# Final validation of the round-2 tree: smoke, full GPU suite, default bench, reference arm.
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/s36_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/s36_gputest.log 2>&1
python bench.py > $O/s36_bench_c3.jsonl 2> $O/s36_bench_c3.err
( time timeout 900 python bench.py --impl reference ) > $O/s36_ref_c3.jsonl 2> $O/s36_ref_c3.err
ls $O | grep s36_
