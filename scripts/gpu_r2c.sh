# round 2 pass c: locality probe, products order experiments, reddit/tiny/sweep on the box harness
R=gpurun_out/r2c; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 600 python -m pytest tests/test_round2_gpu.py -q > $R/pytest_r2.log 2>&1; echo "rc=$?" >> $R/pytest_r2.log
timeout 600 build/probes/request_rate_probe 4 managed > $R/request_rate_locality.jsonl 2>&1
B="python bench.py --config products --steps 20 --warmup 5 --no-cpu --no-e2e"
for v in "" "--plan share=off" "--presort" "--presort --plan share=off" "--plan reorder=on" "--plan reorder=on,share=off" "--plan runs=on"; do
  echo "== $v" >> $R/products_order.log
  timeout 600 $B $v >> $R/products_order.log 2>&1
done
for c in reddit tiny; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $R/bench_$c.json 2> $R/bench_$c.err
done
for rb in 4 16 64 68 128 256 260 400 512 516 1024 2052 2408 4096; do
  timeout 600 python bench.py --config sweep:$rb --steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13 >> $R/bench_sweep.jsonl 2>> $R/bench_sweep.err
done
