# round 2: ut_numa_place + bench --numa replica (one replica per NUMA node)
R=gpurun_out/r2rep; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 1200 python -m pytest tests/test_round2_gpu.py -q -k "numa or replica or box_harness_tiny or islands" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --numa replica > $R/bench_papers_replica1.json 2> $R/bench_papers_replica1.err
