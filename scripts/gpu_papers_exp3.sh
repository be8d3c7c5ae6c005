#!/bin/bash
L=gpurun_out/papers_exp3.log
: > $L
for mb in 24 16 8; do
  echo "== ku1 max_blocks $mb presort" >> $L
  UT_LIB=build/variants/libut_ku1.so UT_MAX_BLOCKS=$mb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --presort --plan reorder=off --max-lists 24 >> $L 2>&1
done
for mb in 74 37 16; do
  echo "== ku1 max_blocks $mb reorder auto" >> $L
  UT_LIB=build/variants/libut_ku1.so UT_MAX_BLOCKS=$mb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
done
for mb in 148 37 16; do
  echo "== ku1 max_blocks $mb products" >> $L
  UT_LIB=build/variants/libut_ku1.so UT_MAX_BLOCKS=$mb timeout 900 python bench.py --config products --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
  echo "== ku1 max_blocks $mb sweep512" >> $L
  UT_LIB=build/variants/libut_ku1.so UT_MAX_BLOCKS=$mb timeout 900 python bench.py --config sweep:512 --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
done
