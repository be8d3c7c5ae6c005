#!/bin/bash
mkdir -p gpurun_out
L=gpurun_out/conc_exp.log
: > $L
for b in 1 2 0; do
  echo "== blocks_per_sm $b quick 1GiB (no reorder)" >> $L
  UT_BLOCKS_PER_SM=$b timeout 600 python scripts/quick_bw.py --table-gib 1 --widths 64,400,512,2408 --plans reorder=off >> $L 2>&1
done
for b in 1 2 0; do
  echo "== blocks_per_sm $b papers" >> $L
  UT_BLOCKS_PER_SM=$b timeout 900 python bench.py --config papers --steps 30 --no-cpu --no-e2e >> $L 2>&1
done
