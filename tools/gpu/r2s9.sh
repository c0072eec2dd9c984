#!/bin/bash
# Same-box A/B of the round-1 final tree (ab_r1) and the current tree on fixed plans
# (env-selected, tuner off) for c1 (temporal blocking), c3 (two plans) and c5.
O=gpurun_out
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s9_${tag}_${tree}.jsonl 2> $O/s9_${tag}_${tree}.err
}
for rep in 1 2; do
  for tree in r1 cur; do
    run c1_$rep $tree c1 LOPE_AUTOTUNE=0
    run c3ded_$rep $tree c3 LOPE_AUTOTUNE=0 LOPE_TILE=1,16,2,8 LOPE_PW=1 LOPE_SHFL=1 LOPE_ZCHUNK=8
    run c3inb_$rep $tree c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64
    run c5inb_$rep $tree c5 LOPE_AUTOTUNE=0 LOPE_TILE=1,8,4,8 LOPE_ZCHUNK=64
  done
  run c1np_$rep cur c1 LOPE_AUTOTUNE=0 LOPE_NVRTC_DEFS=-DLOPE_NO_PAIR
  run c3dednp_$rep cur c3 LOPE_AUTOTUNE=0 LOPE_TILE=1,16,2,8 LOPE_PW=1 LOPE_SHFL=1 LOPE_ZCHUNK=8 LOPE_NVRTC_DEFS=-DLOPE_NO_PAIR
done
ls $O | grep s9_ | wc -l
