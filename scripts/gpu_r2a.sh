# round 2, first pass: build + smoke, round-2 GPU tests, full GPU suite, the new default bench
R=gpurun_out/r2a; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 900 python -m pytest tests/test_round2_gpu.py -q -x > $R/pytest_r2.log 2>&1; echo "rc=$?" >> $R/pytest_r2.log
timeout 1500 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
( time timeout 1200 python bench.py --steps 20 --warmup 5 ) > $R/bench_default.json 2> $R/bench_default.err
timeout 1200 python bench.py --steps 20 --warmup 5 >> $R/bench_default.json 2>> $R/bench_default.err
timeout 900 python bench.py --config products --steps 20 --warmup 5 > $R/bench_products.json 2> $R/bench_products.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > $R/bench_reference.json 2> $R/bench_reference.err
