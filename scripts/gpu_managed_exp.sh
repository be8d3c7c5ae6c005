#!/bin/bash
L=gpurun_out/managed_exp.log
: > $L
for p in "conc=dense" "reorder=off" "conc=sparse"; do
  echo "== papers managed $p" >> $L
  timeout 1200 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 --alloc managed --plan $p >> $L 2>&1
done
for sb in 74 110; do
  echo "== papers managed sparse_blocks $sb" >> $L
  UT_SPARSE_BLOCKS=$sb timeout 1200 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 --alloc managed >> $L 2>&1
done
for c in sweep:512 sweep:64; do
for a in register managed; do
  echo "== $c $a" >> $L
  timeout 1200 python bench.py --config $c --steps 20 --no-cpu --no-e2e --max-lists 24 --alloc $a >> $L 2>&1
  echo "== $c $a reorder=off" >> $L
  timeout 1200 python bench.py --config $c --steps 20 --no-cpu --no-e2e --max-lists 24 --alloc $a --plan reorder=off >> $L 2>&1
done
done
