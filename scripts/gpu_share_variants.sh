#!/bin/bash
# k_share launch variants on products: rows in flight per warp (UT_KU), blocks per SM, load hint.
R=gpurun_out/${1:-sharevar}
mkdir -p $R
A="--steps 30 --no-cpu --no-e2e"
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 600 python bench.py $A > $R/tmp.json 2>> $R/err.log
  python -c "import json; d=json.loads(open('$R/tmp.json').read().strip().splitlines()[-1]); print(json.dumps({'mode':'$label','value':d['value'],'kernel':d['roofline']['achieved'],'plan':d['plan']}))" >> $R/var.jsonl
}
V=build/variants
for rep in 1 2; do
  run base UT_LIB=$V/libut_base.so
  run ku2 UT_LIB=$V/libut_ku2.so
  run ku8 UT_LIB=$V/libut_ku8.so
  run l2_256 UT_LIB=$V/libut_l2_256.so
  run bps1 UT_LIB=$V/libut_base.so UT_BLOCKS_PER_SM=1
  run bps3 UT_LIB=$V/libut_base.so UT_BLOCKS_PER_SM=3
done
