#!/bin/bash
mkdir -p gpurun_out
L=gpurun_out/reorder_exp.log
: > $L
for sh in 21 16 14; do
  echo "== shift $sh products reorder=on" >> $L
  UT_REORDER_SHIFT=$sh timeout 600 python bench.py --config products --steps 50 --no-e2e --no-cpu --plan reorder=on >> $L 2>&1
done
echo "== products reorder=off" >> $L
timeout 600 python bench.py --config products --steps 50 --no-e2e --no-cpu --plan reorder=off >> $L 2>&1
for sh in 21 14; do
  echo "== shift $sh quick 1GiB" >> $L
  UT_REORDER_SHIFT=$sh timeout 600 python scripts/quick_bw.py --table-gib 1 --widths 4,16,64,68,128,256,400 --plans reorder=off,reorder=on >> $L 2>&1
done
