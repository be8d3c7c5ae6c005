# round 2 pass f: in-process coop tests, clock-sampler fix, default repeats
R=gpurun_out/r2f; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py tests/test_coop_gpu.py -q > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err
for i in 1 2 3; do timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 >> $R/bench_default_repeats.jsonl 2>> $R/bench_default.err; done
timeout 900 python bench.py --gpus 2 --oversubscribe --config products --steps 20 --warmup 5 --no-cpu --no-e2e > $R/box2_products.json 2> $R/box2_products.err
timeout 900 python bench.py --gpus 2 --oversubscribe --coop device --config products --steps 20 --warmup 5 --no-cpu > $R/box2_products_coop.json 2> $R/box2_products_coop.err
timeout 900 python bench.py --gpus 4 --oversubscribe --coop device --config reddit --steps 20 --warmup 5 --no-cpu > $R/box4_reddit_coop.json 2> $R/box4_reddit_coop.err
