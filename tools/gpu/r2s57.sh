#!/bin/bash
# Grid-wide producer pacing (LOPE_PACE=<slack planes>): parity, c3/c5 burst and capped, c5 DRAM reads
O=gpurun_out
LOPE_NVRTC_DEFS="-DLOPE_PACE=16" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ragged.py -q -x > $O/s57_tests.log 2>&1
run() {  # tag workload plan defs
  sleep 5
  LOPE_NVRTC_DEFS="$4" timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s57_$1.jsonl 2> $O/s57_$1.err
}
X=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct
for v in 16 4; do
  LOPE_NVRTC_DEFS="-DLOPE_PACE=$v" timeout 600 python tools/ncu_traffic.py --workload c5 --plan 1,8,4,8,0,1,0,0:64 --extra $X \
    | sed "s/^{/{\"pace\": $v, /" >> $O/s57_traffic.jsonl 2>> $O/s57_traffic.err
done
LOPE_NVRTC_DEFS="-DLOPE_PACE=16 -DLOPE_NO_WAIT_TRAP" timeout 600 python tools/ncu_traffic.py --workload c3 --plan 1,16,2,8,0,1,0,0:64 --extra $X \
    | sed "s/^{/{\"pace\": \"16nt\", /" >> $O/s57_traffic.jsonl 2>> $O/s57_traffic.err
for v in base 16 4 32 16nt; do
  D=""; [ $v != base ] && D="-DLOPE_PACE=${v%nt}"; [ $v = 16nt ] && D="$D -DLOPE_NO_WAIT_TRAP"
  run c3inb_$v c3 1,16,2,8,0,1,0,0:64 "$D"
  run c3ded_$v c3 1,16,2,12,1,1,1,0:8 "$D"
  run c5a_$v c5 1,8,4,8,0,1,0,0:64 "$D"
done
