#!/bin/bash
# Round-2 session 3, call 3: multi-array test fix, c4 regression bisect (fp64 dividend
# classification / probe-first waits, interleaved repeats), multi-array producer A/B,
# default c3 bench with the conditional watchdog, one ncu --set full capture of c3.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py -q > $O/s5_ragged.log 2>&1
for rep in 1 2; do
  for v in cur dsetp noprobe both old; do
    d=.; defs=""
    [ $v = dsetp ] && defs="-DLOPE_DIVC_DSETP"
    [ $v = noprobe ] && defs="-DLOPE_NO_PROBE"
    [ $v = both ] && defs="-DLOPE_DIVC_DSETP -DLOPE_NO_PROBE"
    [ $v = old ] && d=ab_old
    (cd $d && LOPE_NVRTC_DEFS="$defs" timeout 300 python bench.py --workload c4 --plan "1,16,4,6,1,0,0,0:1" \
      --steps 20 --warmup 5 --no-e2e --no-cpu --sustained-seconds 1) > $O/s5_c4_${v}_$rep.jsonl 2> $O/s5_c4_${v}_$rep.err
  done
done
timeout 300 python tools/perf_cliffs.py --cases two3d > $O/s5_two3d_pw0.jsonl 2>&1
LOPE_MULTI_PW=1 timeout 300 python tools/perf_cliffs.py --cases two3d > $O/s5_two3d_pw1.jsonl 2>&1
python bench.py > $O/s5_bench_c3.jsonl 2> $O/s5_bench_c3.err
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:^lope_tiled$ --launch-skip 8 -c 1 -o $O/s5_prof_c3_pair -f \
  python bench.py --workload c3 --plan "1,16,2,8,1,1,1,0:8" --steps 12 --warmup 3 --no-e2e --no-cpu \
  --sustained-seconds 0 > $O/s5_ncu_c3.log 2>&1
ls -la $O | tail -5
