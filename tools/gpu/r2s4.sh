#!/bin/bash
# Round-2 session 3, call 2: ragged/rank-1/multi-array parity, their throughput, sustained
# copy bandwidth, and an A/B of the tiled kernel on fixed plans: the tree before the
# probe-first-waits commit (ab_old), the current tree without and with paired fp32 math.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py -q > $O/s4_ragged.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_ragged.py > $O/s4_gputest.log 2>&1
timeout 300 python tools/sustained_copy.py --seconds 3 > $O/s4_copy.jsonl 2> $O/s4_copy.err
timeout 300 python tools/perf_cliffs.py > $O/s4_cliffs.jsonl 2> $O/s4_cliffs.err
for spec in "c3 1,16,2,8,1,0,0,0:64" "c3 1,16,2,8,1,1,1,0:8" "c3 1,8,4,8,1,0,0,0:64" "c4 1,16,4,6,1,0,0,0:1"; do
  set -- $spec
  for tree in old nopair pair; do
    d=.; [ $tree = old ] && d=ab_old
    defs=""; [ $tree = nopair ] && defs="-DLOPE_NO_PAIR"
    tag=$1_$(echo $2 | tr ',:' '__')_$tree
    (cd $d && LOPE_NVRTC_DEFS="$defs" timeout 300 python bench.py --workload $1 --plan "$2" --steps 20 --warmup 5 \
       --no-e2e --no-cpu --sustained-seconds 1.5) > $O/s4_ab_$tag.jsonl 2> $O/s4_ab_$tag.err
  done
done
ls -la $O
