#!/bin/bash
# Plane-loop overhead A/B: sliding single wait, one slot division per plane.
O=gpurun_out
run() {  # tag plan defs
  LOPE_NVRTC_DEFS="$3" timeout 300 python bench.py --workload c3 --plan "$2" --steps 50 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 2 > $O/s35_$1.jsonl 2> $O/s35_$1.err
}
for rep in 1 2; do
  for v in base slide slot both; do
    D=""; [ $v = slide ] && D="-DLOPE_SLIDE_WAIT"; [ $v = slot ] && D="-DLOPE_SLOT_INC"
    [ $v = both ] && D="-DLOPE_SLIDE_WAIT -DLOPE_SLOT_INC"
    run ded_${v}_$rep 1,16,2,12,1,1,1,0:8 "$D"
    run inb_${v}_$rep 1,16,2,8,0,1,0,0:64 "$D"
  done
done
ls $O | grep s35_ | wc -l
