#!/bin/bash
# Decomposition overhead on one GPU: P slabs through the C-ABI communicator (fused
# peer-store steps ordered by stream memory operations, round-robin streams) vs the
# undecomposed domain, config-3-like 7-point fp32, slabs of 512^3.
O=gpurun_out
gcc -O2 -o /tmp/abi_slabs tools/abi_slabs.c -Iinclude -I/usr/local/cuda/include -Lpaper_1502_03504_b200 \
  -llope_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1502_03504_b200 -Wl,-rpath,/usr/local/cuda/lib64
for P in 2 4 8; do
  timeout 300 /tmp/abi_slabs rr $P 512 20 >> $O/s34_slabs.jsonl 2>> $O/s34_slabs.err
done
