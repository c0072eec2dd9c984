#!/bin/bash
O=gpurun_out
for rep in 1 2; do python bench.py > $O/s43_c3_$rep.jsonl 2> $O/s43_c3_$rep.err; done
