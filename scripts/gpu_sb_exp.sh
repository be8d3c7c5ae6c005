#!/bin/bash
L=gpurun_out/sb_exp.log
: > $L
for rep in 1 2; do
for sb in 48 55 64 74 90 110; do
  echo "== sparse_blocks $sb rep $rep" >> $L
  UT_SPARSE_BLOCKS=$sb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
done
done
