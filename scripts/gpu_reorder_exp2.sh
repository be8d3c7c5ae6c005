#!/bin/bash
mkdir -p gpurun_out
L=gpurun_out/reorder_exp2.log
: > $L
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "== products auto" >> $L
timeout 600 python bench.py --config products --steps 50 --no-e2e --no-cpu >> $L 2>&1
echo "== products reorder=on" >> $L
timeout 600 python bench.py --config products --steps 50 --no-e2e --no-cpu --plan reorder=on >> $L 2>&1
echo "== sweep512 auto" >> $L
timeout 600 python bench.py --config sweep:512 --steps 30 --no-e2e --no-cpu >> $L 2>&1
echo "== sweep64 auto" >> $L
timeout 600 python bench.py --config sweep:64 --steps 30 --no-e2e --no-cpu >> $L 2>&1
echo "== quick 1GiB" >> $L
timeout 600 python scripts/quick_bw.py --table-gib 1 --widths 4,16,64,68,128,256 --plans reorder=off,reorder=on >> $L 2>&1
