# round 2: transferred GB/s from the ncu ratios + theoretical link context in the bench line
R=gpurun_out/r2tr; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "box_harness_tiny" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --config products --no-cpu > $R/bench_products.json 2> $R/bench_products.err
