#!/bin/bash
# mbarrier wait loop: no trap counter, longer suspend hint (c3, both plan families, same box)
O=gpurun_out
run() {  # tag workload plan defs
  LOPE_NVRTC_DEFS="$4" timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s53_$1.jsonl 2> $O/s53_$1.err
}
for rep in 1 2; do
  for v in base notrap hint20 both; do
    D=""; [ $v = notrap ] && D="-DLOPE_NO_WAIT_TRAP"; [ $v = hint20 ] && D="-DLOPE_WAIT_HINT_NS=20000"
    [ $v = both ] && D="-DLOPE_NO_WAIT_TRAP -DLOPE_WAIT_HINT_NS=20000"
    run c3ded_${v}_$rep c3 1,16,2,12,1,1,1,0:8 "$D"
    run c3inb_${v}_$rep c3 1,16,2,8,0,1,0,0:64 "$D"
  done
done
