#!/bin/bash
# mbarrier wait variants: trap counter x suspend hint (c3, in-band 64-plane plan), burst and capped
O=gpurun_out
run() {  # tag plan defs
  sleep 5
  LOPE_NVRTC_DEFS="$3" timeout 400 python bench.py --workload c3 --plan "$2" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s56_$1.jsonl 2> $O/s56_$1.err
}
for t in trap notrap; do
  T=""; [ $t = notrap ] && T="-DLOPE_NO_WAIT_TRAP"
  for h in 5000 1000 200 none; do
    H="-DLOPE_WAIT_HINT_NS=$h"; [ $h = none ] && H="-DLOPE_NO_WAIT_HINT"
    run inb_${t}_$h 1,16,2,8,0,1,0,0:64 "$T $H"
  done
done
