#!/bin/bash
L=gpurun_out/blocked_exp.log
: > $L
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
for c in papers sweep:512 sweep:64 sweep:256; do
for conc in sparse dense; do
  echo "== $c conc=$conc" >> $L
  timeout 900 python bench.py --config $c --steps 20 --no-cpu --no-e2e --max-lists 24 --plan conc=$conc >> $L 2>&1
done
done
for sb in 37 55 74 110; do
  echo "== papers sparse_blocks $sb" >> $L
  UT_SPARSE_BLOCKS=$sb timeout 900 python bench.py --config papers --steps 20 --no-cpu --no-e2e --max-lists 24 --plan conc=sparse >> $L 2>&1
done
