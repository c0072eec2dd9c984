#!/bin/bash
# DRAM reads of the no-trap build at full clocks (ncu serialises launches: no power cap)
O=gpurun_out
X=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second
for v in notrap base; do
  D=""; [ $v = notrap ] && D="-DLOPE_NO_WAIT_TRAP"
  for plan in 1,16,2,8,0,1,0,0:64 1,16,2,12,1,1,1,0:8; do
    LOPE_NVRTC_DEFS="$D" timeout 600 python tools/ncu_traffic.py --workload c3 --plan $plan --extra $X \
      | sed "s/^{/{\"variant\": \"$v\", /" >> $O/s55_traffic.jsonl 2>> $O/s55_traffic.err
  done
done
