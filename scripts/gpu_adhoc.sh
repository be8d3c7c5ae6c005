R=gpurun_out/coopsample; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in products reddit; do
  timeout 600 python bench.py --config $c --sample gpu --graph-indptr "hbm,indices=hbm" --coop device --steps 30 --no-cpu --no-e2e --max-lists 16 | sed 's/^{/{"mode": "device", /' >> $R/n1.jsonl 2>> $R/err.log
  for n in 2 4; do
    for m in off device; do
      timeout 900 $TR --nproc-per-node $n --master-port $((29600 + n)) bench.py --gpus $n --backend gloo --config $c --sample gpu --graph-indptr "hbm,indices=hbm" --coop $m --steps 30 --no-cpu --no-e2e --max-lists 16 2>> $R/err.log | grep '^{' | sed "s/^{/{\"mode\": \"$m\", /" >> $R/n$n.jsonl
    done
  done
done
