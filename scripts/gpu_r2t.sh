# round 2 pass t: pipelined GPU sampling in the box harness
R=gpurun_out/r2t; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "pipelined" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
for c in papers products; do
  timeout 900 python bench.py --config $c --sample gpu --pipeline --graph-indptr "hbm,indices=hbm" --steps 20 --warmup 5 --no-cpu --max-lists 25 > $R/bench_${c}_sample_pipeline.json 2> $R/bench_${c}_sample_pipeline.err
done
