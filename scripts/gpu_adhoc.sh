R=gpurun_out/coopart; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_coop_gpu.py -q -x --timeout 300 > $R/pytest.log 2>&1; echo rc=$? >> $R/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --config papers --coop device --alloc managed --steps 30 --no-e2e --max-lists 16 | sed 's/^{/{"mode": "device, managed partitions", /' >> $R/papers.jsonl 2>> $R/err.log
for n in 2 4; do
  timeout 1200 $TR --nproc-per-node $n --master-port $((29700 + n)) bench.py --gpus $n --backend gloo --config papers --coop device --alloc managed --steps 30 --no-cpu --no-e2e --max-lists 16 2>> $R/err.log | grep '^{' | sed "s/^{/{\"mode\": \"device, managed partitions\", /" >> $R/papers.jsonl
  timeout 1200 $TR --nproc-per-node $n --master-port $((29710 + n)) bench.py --gpus $n --backend gloo --config papers --coop off --steps 30 --no-cpu --no-e2e --max-lists 16 2>> $R/err.log | grep '^{' | sed "s/^{/{\"mode\": \"off, shared registered\", /" >> $R/papers.jsonl
done
