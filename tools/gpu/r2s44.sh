#!/bin/bash
# Two-box tiles: parity, c5 plans, and an A/B of the default c3 plans against the
# previous tree (the default instantiations must not move).
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py -q -x -k "two_box or ragged_x_runs" > $O/s44_tests.log 2>&1
run() {  # tag tree workload plan
  local d=.; [ $2 = prev ] && d=ab_prev
  (cd $d && timeout 400 python bench.py --workload $3 --plan "$4" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 2) > $O/s44_$1.jsonl 2> $O/s44_$1.err
}
for rep in 1 2; do
  run c3inb_prev_$rep prev c3 1,16,2,8,0,1,0,0:64
  run c3inb_cur_$rep cur c3 1,16,2,8,0,1,0,0:64
  run c3ded_prev_$rep prev c3 1,16,2,12,1,1,1,0:8
  run c3ded_cur_$rep cur c3 1,16,2,12,1,1,1,0:8
  run c5nb64_$rep cur c5 1,16,2,8,0,1,0,1:64
  run c5w2r4_$rep cur c5 2,8,4,6,0,1,0,0:64
  run c5w2r4nb_$rep cur c5 2,8,4,6,0,1,0,1:64
  run c5w2r2_$rep cur c5 2,8,2,8,0,1,0,0:64
done
ls $O | grep s44_ | wc -l
