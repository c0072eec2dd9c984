#!/bin/bash
# 3-tier stores: same-box A/B vs the round-1 tree (pairs on / off), fixed plans.
O=gpurun_out
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s12_${tag}_${tree}.jsonl 2> $O/s12_${tag}_${tree}.err
}
for rep in 1 2; do
  for tree in r1 cur np; do
    t=$tree; [ $tree = np ] && t=cur
    D=""; [ $tree = np ] && D="-DLOPE_NO_PAIR"
    run c3inb_${rep}_$tree $t c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 LOPE_NVRTC_DEFS="$D"
    run c3ded_${rep}_$tree $t c3 LOPE_AUTOTUNE=0 LOPE_TILE=1,16,2,8 LOPE_PW=1 LOPE_SHFL=1 LOPE_ZCHUNK=8 LOPE_NVRTC_DEFS="$D"
    run c5inb_${rep}_$tree $t c5 LOPE_AUTOTUNE=0 LOPE_TILE=1,8,4,8 LOPE_ZCHUNK=64 LOPE_NVRTC_DEFS="$D"
  done
done
timeout 900 python -m pytest tests/test_gpu_ragged.py tests/test_gpu_parity.py -q -x > $O/s12_tests.log 2>&1
ls $O | grep s12_ | wc -l
