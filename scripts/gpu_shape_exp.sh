#!/bin/bash
L=gpurun_out/shape_exp.log
: > $L
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
for c in papers sweep:64 sweep:512 sweep:2408 sweep:4 products reddit; do
  for conc in auto dense; do
    echo "== $c conc=$conc" >> $L
    timeout 900 python bench.py --config $c --steps 20 --no-cpu --no-e2e --max-lists 24 --plan conc=$conc >> $L 2>&1
  done
done
