#!/bin/bash
# Tiled kernel = round-1 body + compile-time YS (rank 2) / RAG (ragged) instantiations:
# GPU suite, same-box A/B vs round 1, the tuned default bench.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $O/s17_gputest.log 2>&1
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s17_${tag}.jsonl 2> $O/s17_${tag}.err
}
for rep in 1 2; do
  for v in r1 cur; do
    run c3inb_${rep}_$v $v c3 LOPE_AUTOTUNE=0 LOPE_ZCHUNK=64
    run c3ded_${rep}_$v $v c3 LOPE_AUTOTUNE=0 LOPE_TILE=1,16,2,8 LOPE_PW=1 LOPE_SHFL=1 LOPE_ZCHUNK=8
    run c5inb_${rep}_$v $v c5 LOPE_AUTOTUNE=0 LOPE_TILE=1,8,4,8 LOPE_ZCHUNK=64
    run c4_${rep}_$v $v c4 LOPE_AUTOTUNE=0
    run c1_${rep}_$v $v c1 LOPE_AUTOTUNE=0
  done
done
python bench.py --steps 20 --warmup 5 > $O/s17_bench_c3.jsonl 2> $O/s17_bench_c3.err
timeout 300 python tools/perf_cliffs.py > $O/s17_cliffs.jsonl 2>&1
ls $O | grep s17_ | wc -l
