#!/bin/bash
# Tiled kernel rebuilt on the round-1 structure (+ y-streaming, ragged masks, pairs):
# GPU suite, then a same-box A/B against the round-1 tree on fixed plans.
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/s10_gputest.log 2>&1
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s10_${tag}_${tree}.jsonl 2> $O/s10_${tag}_${tree}.err
}
for rep in 1 2; do
  for tree in r1 cur; do
    run c3ded_$rep $tree c3 LOPE_AUTOTUNE=0 LOPE_TILE=1,16,2,8 LOPE_PW=1 LOPE_SHFL=1 LOPE_ZCHUNK=8
    run c3inb_$rep $tree c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64
    run c5inb_$rep $tree c5 LOPE_AUTOTUNE=0 LOPE_TILE=1,8,4,8 LOPE_ZCHUNK=64
    run c4_$rep $tree c4 LOPE_AUTOTUNE=0
    run c1_$rep $tree c1 LOPE_AUTOTUNE=0
  done
done
ls $O | grep s10_ | wc -l
