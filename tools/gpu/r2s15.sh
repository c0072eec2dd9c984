#!/bin/bash
# Store state rebuilt in cold paths only: same-box A/B vs round 1 (fixed plans), then the
# default c3 bench (pipelined e2e batch).
O=gpurun_out
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s15_${tag}.jsonl 2> $O/s15_${tag}.err
}
for rep in 1 2; do
  for v in r1 cur np; do
    t=$v; [ $v = np ] && t=cur
    D=""; [ $v = np ] && D="-DLOPE_NO_PAIR"
    run c3inb_${rep}_$v $t c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64 LOPE_NVRTC_DEFS="$D"
    run c3ded_${rep}_$v $t c3 LOPE_AUTOTUNE=0 LOPE_TILE=1,16,2,8 LOPE_PW=1 LOPE_SHFL=1 LOPE_ZCHUNK=8 LOPE_NVRTC_DEFS="$D"
    run c5inb_${rep}_$v $t c5 LOPE_AUTOTUNE=0 LOPE_TILE=1,8,4,8 LOPE_ZCHUNK=64 LOPE_NVRTC_DEFS="$D"
  done
done
python bench.py --steps 20 --warmup 5 > $O/s15_bench_c3.jsonl 2> $O/s15_bench_c3.err
ls $O | grep s15_ | wc -l
