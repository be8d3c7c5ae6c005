# round 2, last session: tables share per-device scratch pool + error-word slab (no CUDA
# allocation per table); the full GPU suite, smoke, the pool probe, and the bench default
R=gpurun_out/r2pool2; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 900 python scripts/pool_probe.py > $R/pool_probe.jsonl 2> $R/pool_probe.err
timeout 2400 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
