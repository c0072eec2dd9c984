#!/bin/bash
# Validation of the current tree: smoke, full GPU suite, default bench.
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/s28_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/s28_gputest.log 2>&1
python bench.py > $O/s28_bench_c3.jsonl 2> $O/s28_bench_c3.err
ls $O | grep s28_
