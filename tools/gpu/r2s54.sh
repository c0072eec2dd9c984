#!/bin/bash
# Per-step time series of the in-band plan with and without the wait-loop trap counter
O=gpurun_out
for v in base notrap base notrap; do
  D=""; [ $v = notrap ] && D="-DLOPE_NO_WAIT_TRAP"
  sleep 10
  LOPE_NVRTC_DEFS="$D" LOPE_ZCHUNK=64 N=2000 timeout 300 python tools/probe_power.py >> $O/s54_$v.jsonl 2>> $O/s54_$v.err
done
