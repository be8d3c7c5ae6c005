# round 2 pass x: ut_numa_interleave (test + papers A/B on node 0), reddit repeats (r2w's reddit
# ran while the host's DRAM read and memcpy ceilings had dropped: 64.9 GB/s, 51.2 after timing)
R=gpurun_out/r2x; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 600 python -m pytest tests/test_round2_gpu.py -q -k numa > $R/pytest_numa.log 2>&1; echo "rc=$?" >> $R/pytest_numa.log
B="python3 bench.py --gpus 1 --steps 20 --warmup 5"
for i in 1 2; do
  timeout 900 $B --numa interleave >> $R/bench_papers_numa.jsonl 2>> $R/bench.err
  timeout 900 $B >> $R/bench_papers_default.jsonl 2>> $R/bench.err
  timeout 900 $B --config reddit >> $R/bench_reddit.jsonl 2>> $R/bench.err
done
