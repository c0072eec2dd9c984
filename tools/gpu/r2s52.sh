#!/bin/bash
# Validation on a fresh box with the pruned cubin cache: smoke, GPU suite, default bench, reference arm
O=gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/s52_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/s52_gputest.log 2>&1
timeout 900 python bench.py > $O/s52_bench_c3.jsonl 2> $O/s52_bench_c3.err
timeout 900 python bench.py --impl reference > $O/s52_ref_c3.jsonl 2> $O/s52_ref_c3.err
