#!/bin/bash
# Streaming (evict-first) output stores vs plain: c3 / c5 time and c5 DRAM reads
O=gpurun_out
run() {  # tag workload plan defs
  LOPE_NVRTC_DEFS="$4" timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s50_$1.jsonl 2> $O/s50_$1.err
}
X=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct
LOPE_NVRTC_DEFS="-DLOPE_ST_CS" timeout 600 python tools/ncu_traffic.py --workload c5 --plan 1,8,4,8,0,1,0,0:64 --extra $X >> $O/s50_traffic.jsonl 2>> $O/s50_traffic.err
timeout 600 python tools/ncu_traffic.py --workload c5 --plan 1,8,4,8,0,1,0,0:64 --extra $X >> $O/s50_traffic.jsonl 2>> $O/s50_traffic.err
LOPE_NVRTC_DEFS="-DLOPE_ST_CS" timeout 600 python tools/ncu_traffic.py --workload c3 --plan 1,16,2,8,0,1,0,0:64 --extra $X >> $O/s50_traffic.jsonl 2>> $O/s50_traffic.err
for rep in 1 2; do
  for v in base cs; do
    D=""; [ $v = cs ] && D="-DLOPE_ST_CS"
    run c3inb_${v}_$rep c3 1,16,2,8,0,1,0,0:64 "$D"
    run c3ded_${v}_$rep c3 1,16,2,12,1,1,1,0:8 "$D"
    run c5a_${v}_$rep c5 1,8,4,8,0,1,0,0:64 "$D"
    run c5b_${v}_$rep c5 1,16,2,8,0,1,0,1:64 "$D"
  done
done
