#!/bin/bash
# Config 3 plans over a long capped window: energy per point decides the sustained rate
O=gpurun_out
run() {  # tag plan
  sleep 10
  timeout 400 python bench.py --workload c3 --plan "$2" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 6 > $O/s65_$1.jsonl 2> $O/s65_$1.err
}
for rep in 1 2; do
  run inb1648_$rep 1,8,4,8,0,1,0,0:64
  run inb1628_$rep 1,16,2,8,0,1,0,0:64
  run ded12z8_$rep 1,16,2,12,1,1,1,0:8
  run inb1648nb_$rep 1,8,4,8,0,1,0,1:64
done
