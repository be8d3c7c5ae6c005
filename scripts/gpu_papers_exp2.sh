#!/bin/bash
L=gpurun_out/papers_exp2.log
: > $L
for v in base ku2 ku1; do
  for mb in 148 74 37; do
    echo "== $v max_blocks $mb presort" >> $L
    UT_LIB=build/variants/libut_$v.so UT_MAX_BLOCKS=$mb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --presort --plan reorder=off --max-lists 24 >> $L 2>&1
  done
done
