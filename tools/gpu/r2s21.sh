#!/bin/bash
# Drop-in Machine throughput vs the reference Machine; c3 tile experiments (fixed plans).
O=gpurun_out
timeout 900 python tools/machine_bench.py > $O/s21_machine.jsonl 2> $O/s21_machine.err
run() {  # tag workload plan
  timeout 300 python bench.py --workload $2 --plan "$3" --steps 50 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 1 > $O/s21_$1.jsonl 2> $O/s21_$1.err
}
for rep in 1 2; do
  run c3_inb28_z64_$rep c3 1,16,2,8,0,1,0,0:64
  run c3_inb46_z64_$rep c3 1,16,4,6,0,1,0,0:64
  run c3_inb46_z32_$rep c3 1,16,4,6,0,1,0,0:32
  run c3_ded212_z8_$rep c3 1,16,2,12,1,1,1,0:8
done
ls $O | grep s21_ | wc -l
