# round 2 pass l: e2e noise after the scratch growth fix
R=gpurun_out/r2l; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "gather_host" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
for i in 1 2 3 4; do UT_BENCH_DEBUG=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-check >> $R/e2e_noise.jsonl 2>> $R/e2e_noise.err; done
