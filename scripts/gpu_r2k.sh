# round 2 pass k: e2e noise check
R=gpurun_out/r2k; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
for i in 1 2 3 4; do UT_BENCH_DEBUG=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-check >> $R/e2e_noise.jsonl 2>> $R/e2e_noise.err; done
