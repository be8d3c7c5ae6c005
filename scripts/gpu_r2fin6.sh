# round 2, last session: final verification at HEAD (driver order) after the recycling allocator
# and the per-device shared table resources, plus the N>1 harness on this one GPU (oversubscribed)
R=gpurun_out/r2fin6; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --config products > $R/bench_products.json 2> $R/bench_products.err
timeout 600 python3 bench.py --gpus 2 --oversubscribe --steps 5 --warmup 3 --config products > $R/box2_products.json 2> $R/box2_products.err
timeout 600 python3 bench.py --gpus 4 --oversubscribe --coop device --steps 5 --warmup 3 --config reddit > $R/box4_reddit_coop.json 2> $R/box4_reddit_coop.err
