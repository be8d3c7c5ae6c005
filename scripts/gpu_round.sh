#!/bin/bash
# Full measurement pass: build, smoke, GPU parity tests, bench lines for every config, the
# reference arm, ncu launch lists and one full ncu capture. Everything lands in gpurun_out/R/.
R=gpurun_out/${1:-round}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
timeout 900 python bench.py > $R/bench_default.json 2> $R/bench_default.err
timeout 900 python bench.py --impl reference --steps 10 > $R/bench_reference.json 2> $R/bench_reference.err
for c in reddit papers tiny; do
  timeout 1200 python bench.py --config $c --steps 50 > $R/bench_$c.json 2> $R/bench_$c.err
done
for rb in 4 8 16 32 64 68 100 128 256 400 512 1024 1372 2048 2052 2408 4096; do
  timeout 600 python bench.py --config sweep:$rb --steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13 >> $R/bench_sweep.jsonl 2>> $R/bench_sweep.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_products.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_papers.csv python bench.py --config papers --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 4 -c 1 -o $R/prof_products python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > $R/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 4 -c 1 -o $R/prof_papers python bench.py --config papers --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > $R/ncu_full_papers.log 2>&1
