#!/bin/bash
L=gpurun_out/pf_exp.log
: > $L
for pf in 0 256 1024 4096; do
  for sb in 37 74; do
    echo "== pf $pf sparse_blocks $sb" >> $L
    UT_PF_DIST=$pf UT_SPARSE_BLOCKS=$sb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
  done
done
for sb in 30 45 55; do
  echo "== pf 0 sparse_blocks $sb" >> $L
  UT_SPARSE_BLOCKS=$sb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
done
