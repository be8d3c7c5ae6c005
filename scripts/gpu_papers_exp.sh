#!/bin/bash
L=gpurun_out/papers_exp.log
: > $L
echo "== presort, reorder off, 1 blk/SM" >> $L
UT_BLOCKS_PER_SM=1 timeout 900 python bench.py --config papers --steps 30 --no-cpu --no-e2e --presort --plan reorder=off >> $L 2>&1
echo "== presort, reorder off, full" >> $L
timeout 900 python bench.py --config papers --steps 30 --no-cpu --no-e2e --presort --plan reorder=off >> $L 2>&1
echo "== shift 23 (auto), 1 blk" >> $L
UT_BLOCKS_PER_SM=1 timeout 900 python bench.py --config papers --steps 30 --no-cpu --no-e2e >> $L 2>&1
