# round 2 pass e: full verification at HEAD (smoke, every GPU test, bench lines, sweep)
R=gpurun_out/r2e; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 1800 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
for i in 1 2; do timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 >> $R/bench_default_repeats.jsonl 2>> $R/bench_default.err; done
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err
for c in products reddit; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $R/bench_$c.json 2> $R/bench_$c.err; done
for rb in 4 8 16 32 64 68 100 128 132 256 260 400 512 516 1024 1028 1172 1372 2048 2052 2064 2076 2408 3200 4092 4096; do
  timeout 600 python bench.py --config sweep:$rb --steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13 >> $R/bench_sweep.jsonl 2>> $R/bench_sweep.err
done
