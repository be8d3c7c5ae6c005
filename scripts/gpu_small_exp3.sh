#!/bin/bash
# Small rows over the 16-GiB sweep table: launch shape (sparse grid size, dense) vs run merge.
R=gpurun_out/${1:-small3}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
A="--steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13"
for rb in 64 128; do
  for b in 37 110 148 296 592; do
    UT_SPARSE_BLOCKS=$b timeout 600 python bench.py --config sweep:$rb $A > $R/tmp.json 2>> $R/err.log
    python -c "import json,sys; d=json.loads(open('$R/tmp.json').read().strip().splitlines()[-1]); print(json.dumps({'rb':$rb,'mode':'sparse$b','value':d['value'],'kernel':d['roofline']['achieved']}))" >> $R/shape.jsonl
  done
  timeout 600 python bench.py --config sweep:$rb $A --plan conc=dense > $R/tmp.json 2>> $R/err.log
  python -c "import json,sys; d=json.loads(open('$R/tmp.json').read().strip().splitlines()[-1]); print(json.dumps({'rb':$rb,'mode':'dense','value':d['value'],'kernel':d['roofline']['achieved']}))" >> $R/shape.jsonl
  timeout 600 python bench.py --config sweep:$rb $A --plan runs=on > $R/tmp.json 2>> $R/err.log
  python -c "import json,sys; d=json.loads(open('$R/tmp.json').read().strip().splitlines()[-1]); print(json.dumps({'rb':$rb,'mode':'runs','value':d['value'],'kernel':d['roofline']['achieved']}))" >> $R/shape.jsonl
done
