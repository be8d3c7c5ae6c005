#!/bin/bash
# Small rows over the 16-GiB sweep table: bucket order vs row order inside buckets (UT_REORDER_EXACT
# was a temporary A/B knob that ran k_bucket_sort after the scatter; removed after this run).
R=gpurun_out/${1:-small2}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
A="--steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13"
for rb in 16 64 128 256 400; do
  timeout 600 python bench.py --config sweep:$rb $A >> $R/default.jsonl 2>> $R/err.log
  UT_REORDER_EXACT=1 timeout 600 python bench.py --config sweep:$rb $A >> $R/exact.jsonl 2>> $R/err.log
  UT_REORDER_EXACT=1 UT_REORDER_SHIFT=21 timeout 600 python bench.py --config sweep:$rb $A >> $R/exact21.jsonl 2>> $R/err.log
done
UT_REORDER_EXACT=1 timeout 900 python bench.py --config papers --alloc register --steps 20 --no-cpu --no-e2e >> $R/papers_reg_exact.jsonl 2>> $R/err.log
