#!/bin/bash
# Final tree as the driver runs it: smoke, default bench at K=20 W=5, reference arm
O=gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/s67_smoke.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/s67_bench_c3.jsonl 2> $O/s67_bench_c3.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/s67_ref_c3.jsonl 2> $O/s67_ref_c3.err
