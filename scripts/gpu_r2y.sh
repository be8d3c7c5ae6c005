# round 2 pass y: ut_numa_interleave — placement read back (test); the bench's record when the
# driver does not apply host-NUMA placement (--numa interleave on this pool's one-node boxes)
R=gpurun_out/r2y; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 600 python -m pytest tests/test_round2_gpu.py -q > $R/pytest_r2.log 2>&1; echo "rc=$?" >> $R/pytest_r2.log
timeout 600 python scripts/numa_probe.py > $R/numa_probe.jsonl 2> $R/numa_probe.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --numa interleave --no-cpu > $R/bench_numa.json 2> $R/bench_numa.err
