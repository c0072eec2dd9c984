#!/bin/bash
# c1 after the small-field y-chunk fix (default bench, and A/B vs round 1), c3 default x3.
O=gpurun_out
run() {  # tag tree workload env...
  local tag=$1 tree=$2 wl=$3; shift 3
  local d=.; [ $tree = r1 ] && d=ab_r1
  (cd $d && env "$@" timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu \
     $( [ $tree = r1 ] || echo --sustained-seconds 0 )) > $O/s20_${tag}.jsonl 2> $O/s20_${tag}.err
}
python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu > $O/s20_c1_default.jsonl 2> $O/s20_c1_default.err
for rep in 1 2; do
  run c1_${rep}_r1 r1 c1 LOPE_AUTOTUNE=0
  run c1_${rep}_cur cur c1 LOPE_AUTOTUNE=0
  run c1nt_${rep}_r1 r1 c1 LOPE_AUTOTUNE=0 LOPE_NO_TBLOCK=1
  run c1nt_${rep}_cur cur c1 LOPE_AUTOTUNE=0 LOPE_NO_TBLOCK=1
done
for rep in 1 2 3; do
  python bench.py --no-cpu > $O/s20_c3_$rep.jsonl 2> $O/s20_c3_$rep.err
done
ls $O | grep s20_ | wc -l
