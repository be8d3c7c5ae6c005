# round 2: ut_gather_host output-range walk (islands around an unpinned gap -> copy-engine path)
R=gpurun_out/r2hr; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py tests/test_gather_gpu.py -q -k "gather_host" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
