# round 2: the CPU-centric baseline at k GPUs (cores/k threads per GPU, all at once)
R=gpurun_out/r2pyk; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "cpu_baseline_at_two_gpus or two_workers_one_gpu or box_harness_tiny" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
