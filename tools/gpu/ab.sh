#!/bin/bash
# A/B of tiled-kernel changes on fixed plans (no tuning): bench timing (20-step window and a
# 2 s sustained window) and ncu counters of the lope_tiled launches.
#   bash tools/gpu/ab.sh TAG "WL PLAN [DEFS]" ...
O=gpurun_out
TAG=$1; shift
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
i=0
for spec in "$@"; do
  set -- $spec
  WL=$1; PLAN=$2; DEFS=${3:-}
  i=$((i+1))
  export LOPE_NVRTC_DEFS="$DEFS"
  python bench.py --workload $WL --plan "$PLAN" --steps 20 --warmup 5 --no-e2e --no-cpu --sustained-seconds 2 \
    > $O/ab_${TAG}_$i.jsonl 2> $O/ab_${TAG}_$i.err
  /usr/local/cuda/bin/ncu --metrics $M --cache-control none --clock-control none -k regex:^lope_tiled$ \
    --launch-skip 8 -c 3 --csv --log-file $O/ab_${TAG}_$i.csv \
    python bench.py --workload $WL --plan "$PLAN" --steps 14 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 \
    > /dev/null 2> $O/ab_${TAG}_$i.ncu.err
  echo "$i $WL $PLAN $DEFS" >> $O/ab_${TAG}_index.txt
done
