#!/bin/bash
L=gpurun_out/alloc_exp.log
: > $L
timeout 900 python -m pytest tests/test_gather_gpu.py -x -q -m gpu -k create > gpurun_out/pytest_create.log 2>&1
for c in products papers; do
for a in register pinned managed vmm; do
  echo "== $c alloc=$a" >> $L
  timeout 1200 python bench.py --config $c --steps 20 --no-cpu --max-lists 24 --alloc $a >> $L 2>&1
done
done
