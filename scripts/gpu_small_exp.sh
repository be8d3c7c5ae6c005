#!/bin/bash
# Small rows over the 16-GiB sweep table: bucket reorder (default) vs exact order (runs=on) vs
# 2-MiB buckets (UT_REORDER_SHIFT=21).
R=gpurun_out/${1:-small}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
A="--steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13"
for rb in 16 64 128; do
  timeout 600 python bench.py --config sweep:$rb $A >> $R/default.jsonl 2>> $R/err.log
  timeout 600 python bench.py --config sweep:$rb $A --plan runs=on >> $R/runs.jsonl 2>> $R/err.log
  UT_REORDER_SHIFT=21 timeout 600 python bench.py --config sweep:$rb $A >> $R/shift21.jsonl 2>> $R/err.log
  UT_REORDER_SHIFT=14 timeout 600 python bench.py --config sweep:$rb $A >> $R/shift14.jsonl 2>> $R/err.log
done
