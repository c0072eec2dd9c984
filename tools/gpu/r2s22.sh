#!/bin/bash
# c3 under the power cap: fewer resident CTAs (LOPE_GRID) and the unrolled plane loop.
O=gpurun_out
run() {  # tag plan env...
  local tag=$1 plan=$2; shift 2
  env "$@" timeout 300 python bench.py --workload c3 --plan "$plan" --steps 50 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 2 > $O/s22_$tag.jsonl 2> $O/s22_$tag.err
}
for rep in 1 2; do
  for gr in 147 131 113 97; do
    run ded_g${gr}_$rep 1,16,2,12,1,1,1,0:8 LOPE_GRID=$gr
  done
  run inb_$rep 1,16,2,8,0,1,0,0:64
  run inb_u2_$rep 1,16,2,8,0,1,0,0:64 LOPE_NVRTC_DEFS=-DLOPE_UNROLL2
  run ded_u2_$rep 1,16,2,12,1,1,1,0:8 LOPE_NVRTC_DEFS=-DLOPE_UNROLL2
done
ls $O | grep s22_ | wc -l
