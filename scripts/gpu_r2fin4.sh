# round 2, re-entry session: full verification at HEAD final: after the k-GPU CPU baseline, host_links, transferred GB/s, managed full-size and 2^31-row tests (driver-like order)
R=gpurun_out/r2fin4; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --config products > $R/bench_products.json 2> $R/bench_products.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --config reddit > $R/bench_reddit.json 2> $R/bench_reddit.err
