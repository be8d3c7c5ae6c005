#!/bin/bash
L=gpurun_out/shape_exp2.log
: > $L
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
for c in papers sweep:64 sweep:512 sweep:2408 sweep:4 sweep:256 sweep:128; do
  echo "== $c auto" >> $L
  timeout 900 python bench.py --config $c --steps 20 --no-cpu --no-e2e --max-lists 24 >> $L 2>&1
done
