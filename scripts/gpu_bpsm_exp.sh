#!/bin/bash
L=gpurun_out/bpsm_exp.log
: > $L
for b in 1 2 0; do
for c in sweep:64 sweep:256 sweep:2408 papers products; do
  echo "== bpsm $b $c" >> $L
  UT_BLOCKS_PER_SM=$b timeout 900 python bench.py --config $c --steps 20 --no-cpu --no-e2e --max-lists 16 >> $L 2>&1
done
done
for ip in host hbm; do
  echo "== pipeline products indptr=$ip bpsm1" >> $L
  UT_BLOCKS_PER_SM=1 timeout 900 python bench.py --config products --sample gpu --pipeline --graph-indptr $ip --steps 30 --max-lists 16 --no-cpu >> $L 2>&1
done
