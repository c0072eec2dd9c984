#!/bin/bash
# Round-2 session 3, call 4: GPU suites after the multi-array producer change, c4 bisect
# across old (939676e) / mid (8aec943) / cur, multi-array throughput.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py tests/test_gpu_parity.py -q -x > $O/s6_tests.log 2>&1
for rep in 1 2; do
  for v in old mid cur; do
    d=.; [ $v = old ] && d=ab_old; [ $v = mid ] && d=ab_mid
    (cd $d && timeout 300 python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:1" \
      --steps 20 --warmup 5 --no-e2e --no-cpu --sustained-seconds 1) > $O/s6_c4_${v}_$rep.jsonl 2> $O/s6_c4_${v}_$rep.err
  done
done
timeout 300 python tools/perf_cliffs.py --cases two3d,ragged3d,rank1 > $O/s6_cliffs.jsonl 2>&1
ls -la $O | tail -3
