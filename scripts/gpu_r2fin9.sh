# round 2, last session: verification at HEAD after the last-table scratch trim (driver order)
R=gpurun_out/r2fin9; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --config products > $R/bench_products.json 2> $R/bench_products.err
