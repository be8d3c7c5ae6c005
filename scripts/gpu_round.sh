#!/bin/bash
# Full measurement pass: build, smoke, GPU parity tests, bench lines for every config, the
# reference arm, GPU-sampling lines, repeat runs of the default line, ncu launch lists and full
# captures of the gather kernel. Everything lands in gpurun_out/R/.
R=gpurun_out/${1:-round}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
for i in 1 2 3 4 5; do
  timeout 900 python bench.py >> $R/bench_default_repeats.jsonl 2>> $R/bench_default.err
done
tail -n 1 $R/bench_default_repeats.jsonl > $R/bench_default.json
timeout 900 python bench.py --impl reference > $R/bench_reference.json 2> $R/bench_reference.err
for c in reddit papers tiny; do
  timeout 1200 python bench.py --config $c --steps 50 > $R/bench_$c.json 2> $R/bench_$c.err
done
timeout 1200 python bench.py --config papers --alloc register --steps 50 --no-cpu > $R/bench_papers_registered.json 2>> $R/bench_papers.err
for rb in 4 8 16 32 64 68 100 128 256 400 512 1024 1372 2048 2052 2408 4096; do
  timeout 600 python bench.py --config sweep:$rb --steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13 >> $R/bench_sweep.jsonl 2>> $R/bench_sweep.err
done
for c in products papers; do
  timeout 900 python bench.py --config $c --sample gpu --graph --graph-indptr "hbm,indices=hbm" --steps 30 --no-cpu --max-lists 16 >> $R/bench_gpu_sampling.jsonl 2>> $R/bench_gpu_sampling.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_products.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_papers.csv python bench.py --config papers --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 4 -c 1 -o $R/prof_products python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > $R/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 4 -c 1 -o $R/prof_papers python bench.py --config papers --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > $R/ncu_full_papers.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_multi -s 4 -c 1 -o $R/prof_reddit python bench.py --config reddit --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > $R/ncu_full_reddit.log 2>&1
