#!/bin/bash
# Functional check of bench.py's N>1 path on a one-GPU box: 2 ranks share the device
# (gloo for the setup records; the communicator falls back to host ordering). Not a
# measurement.
O=gpurun_out
for wl in c3 c4; do
  LOPE_BENCH_BACKEND=gloo timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload $wl --steps 4 --warmup 3 \
    --no-cpu --no-e2e --sustained-seconds 0 > $O/s27_n2_$wl.jsonl 2> $O/s27_n2_$wl.err
  echo "$wl rc=$?" >> $O/s27_rc.txt
done
nvidia-smi --query-gpu=name,utilization.gpu --format=csv >> $O/s27_rc.txt
