# round 2 pass i: verify gather_host change, e2e repeats
R=gpurun_out/r2i; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 1200 python -m pytest tests/test_round2_gpu.py tests/test_gather_gpu.py -q > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
for i in 1 2 3; do timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 >> $R/bench_default_repeats.jsonl 2>> $R/bench_default.err; done
