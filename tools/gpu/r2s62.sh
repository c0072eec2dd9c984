#!/bin/bash
# Short z-chunks with y-banded unit walks on c5 (z-halo planes reused while the band's
# next chunk runs in the same wave)
O=gpurun_out
run() {  # tag workload plan
  sleep 5
  timeout 400 python bench.py --workload $2 --plan "$3" --steps 20 --warmup 5 --no-e2e --no-cpu \
    --sustained-seconds 3 > $O/s62_$1.jsonl 2> $O/s62_$1.err
}
run c5_inb c5 1,8,4,8,0,1,0,0:64
for yb in 2 4 8; do run c5_d12z8yb$yb c5 1,16,2,12,1,1,1,0:8:$yb; done
run c5_d12z16yb4 c5 1,16,2,12,1,1,1,0:16:4
run c5_inbz16yb4 c5 1,8,4,8,0,1,0,0:16:4
run c5_inbz32yb4 c5 1,8,4,8,0,1,0,0:32:4
for yb in 4 8; do run c3_d12z8yb$yb c3 1,16,2,12,1,1,1,0:8:$yb; done
run c3_d12z8 c3 1,16,2,12,1,1,1,0:8
