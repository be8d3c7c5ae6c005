# round 2 pass h: e2e host->host variants on the papers-shaped managed table
R=gpurun_out/r2h; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-check"
for v in "UT_HOST_CHUNK=8388608" "UT_HOST_CHUNK=2097152" "UT_HOST_CHUNK=4194304" "UT_HOST_CHUNK=16777216" "UT_HOST_CHUNK=33554432" "UT_HOST_CHUNK=67108864" "UT_HOST_DIRECT=1" "UT_HOST_DIRECT=1 UT_MAX_BLOCKS=148"; do
  echo "== $v" >> $R/e2e_variants.log
  env $v timeout 600 $B >> $R/e2e_variants.log 2>&1
done
