R=gpurun_out/tohbm2; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
UT_BENCH_DEBUG=1 timeout 600 python bench.py --config reddit --steps 50 --no-cpu > $R/bench_reddit.json 2> $R/bench_reddit.err
