#!/bin/bash
# Cooperative gather (ut_coop) vs independent gathers: N ranks as processes sharing this box's
# one GPU and its one host link (the "shared host link" case of SURVEY NEXT-4 (ii)).
R=gpurun_out/${1:-coop_bench}; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in products reddit papers; do
  timeout 600 python bench.py --config $c --coop device --steps 30 --no-cpu --no-e2e --max-lists 16 >> $R/coop_n1.jsonl 2>> $R/err.log
  for n in 2 4; do
    for m in off device host; do
      timeout 900 $TR --nproc-per-node $n --master-port $((29500 + n)) bench.py --gpus $n --backend gloo --config $c --coop $m --steps 30 --no-cpu --no-e2e --max-lists 16 2>> $R/err.log | grep '^{' | sed "s/^{/{\"mode\": \"$m\", /" >> $R/coop_n$n.jsonl
    done
  done
done
