#!/bin/bash
O=gpurun_out
for rep in 1 2 3; do python bench.py > $O/s42_c3_$rep.jsonl 2> $O/s42_c3_$rep.err; done
