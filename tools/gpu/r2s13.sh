#!/bin/bash
# Bisect the in-band plan's slowdown vs round 1: pairs, LopeVecOut stores.
O=gpurun_out
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s13_${tag}.jsonl 2> $O/s13_${tag}.err
}
for rep in 1 2; do
  run c3inb_${rep}_r1 r1 c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64
  run c3inb_${rep}_cur cur c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64
  run c3inb_${rep}_np cur c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 LOPE_NVRTC_DEFS=-DLOPE_NO_PAIR
  run c3inb_${rep}_os cur c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 LOPE_NVRTC_DEFS=-DLOPE_OLD_STORE
  run c3inb_${rep}_npos cur c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 "LOPE_NVRTC_DEFS=-DLOPE_NO_PAIR -DLOPE_OLD_STORE"
done
ls $O | grep s13_ | wc -l
