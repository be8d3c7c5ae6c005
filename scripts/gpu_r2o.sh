# round 2 pass o: GPU sampling in the box harness
R=gpurun_out/r2o; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 1800 python -m pytest tests/test_round2_gpu.py -q -k "sampling" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python bench.py --sample gpu --config products --steps 20 --warmup 5 --no-cpu --graph-indptr "hbm,indices=hbm" > $R/bench_products_sample.json 2> $R/bench_products_sample.err
timeout 900 python bench.py --sample gpu --config papers --steps 20 --warmup 5 --no-cpu --graph-indptr "hbm,indices=hbm" > $R/bench_papers_sample.json 2> $R/bench_papers_sample.err
