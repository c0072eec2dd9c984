#!/bin/bash
# Ragged tier check, throughput of the former cliffs, DRAM traffic per plan (the plans the
# tuner picks on c2-c5) for roofline.traffic, and a launch list of the default bench.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py -q -x > $O/s18_ragged.log 2>&1
timeout 300 python tools/perf_cliffs.py > $O/s18_cliffs.jsonl 2>&1
for spec in "c3 1,16,2,8,0,1,0,0:64" "c3 1,16,2,8,0,1,0,0:32" "c3 1,16,2,12,1,1,1,0:8" "c3 1,16,2,8,1,1,1,0:8" \
            "c3 1,16,2,10,1,1,1,0:6" "c4 1,16,4,6,0,1,0,0:8" "c4 1,16,4,6,1,1,0,0:8" "c2 1,16,2,8,1,1,0,0:8" \
            "c2 1,16,2,12,1,1,0,0:8" "c5 1,16,2,8,0,1,0,0:32" "c5 1,16,2,8,0,1,0,1:64" "c5 1,8,4,8,0,1,0,0:64"; do
  set -- $spec
  timeout 600 python tools/ncu_traffic.py --workload $1 --plan "$2" >> $O/s18_traffic.jsonl 2>> $O/s18_traffic.err
done
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/s18_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 \
  > $O/s18_launches_c3.log 2>&1
ls $O | grep s18_
