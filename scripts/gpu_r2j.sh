# round 2 pass j: e2e (direct host stores) launch-shape variants on papers
R=gpurun_out/r2j; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-check"
for v in "X=1" "UT_BLOCKS_PER_SM=1" "UT_BLOCKS_PER_SM=4" "UT_BLOCKS_PER_SM=0" "UT_MAX_BLOCKS=74" "X=stage"; do
  echo "== $v" >> $R/e2e_shape.log
  if [ "$v" = "X=stage" ]; then timeout 600 $B --plan stage=on >> $R/e2e_shape.log 2>&1; else env $v timeout 600 $B >> $R/e2e_shape.log 2>&1; fi
done
