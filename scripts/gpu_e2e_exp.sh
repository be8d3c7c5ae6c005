#!/bin/bash
# Host->host e2e (ut_gather_host) on products: direct stores vs copy-engine pipeline, each with
# the gather grid capped (UT_MAX_BLOCKS) to leave the upstream direction room for the writes.
R=gpurun_out/${1:-e2e}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 600 python bench.py --steps 20 --no-cpu > $R/tmp.json 2>> $R/err.log
  python -c "import json; d=json.loads(open('$R/tmp.json').read().strip().splitlines()[-1]); print(json.dumps({'mode':'$label','value':d['value'],'e2e':d['e2e']['value'],'to_hbm':d['e2e']['to_hbm']['value']}))" >> $R/e2e.jsonl
}
run direct X=1
for b in 148 74 37 18; do run direct_b$b UT_MAX_BLOCKS=$b; done
run pipe8M UT_HOST_PIPELINE=1
for b in 148 74 37; do run pipe8M_b$b UT_HOST_PIPELINE=1 UT_MAX_BLOCKS=$b; done
run pipe32M UT_HOST_PIPELINE=1 UT_HOST_CHUNK=33554432
run pipe32M_b74 UT_HOST_PIPELINE=1 UT_HOST_CHUNK=33554432 UT_MAX_BLOCKS=74
run pipe2M UT_HOST_PIPELINE=1 UT_HOST_CHUNK=2097152
