# round 2: maximum-size gathers (n > 2^31 rows)
R=gpurun_out/r2max; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 1500 python -m pytest tests/test_round2_gpu.py -q -k beyond_2pow31 > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
