# round 2 pass s: GPU sampling pipelined with the gather, CSR in HBM
R=gpurun_out/r2s; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
for c in products papers; do
  for v in "" "--pipeline"; do
    echo "== $c $v" >> $R/sample_pipeline.log
    timeout 900 python bench.py --config $c --sample gpu --graph-indptr "hbm,indices=hbm" --steps 20 --warmup 5 --no-cpu --max-lists 25 $v >> $R/sample_pipeline.log 2>&1
  done
done
