# round 2: full-size parity on the managed table (the bench default's table memory)
R=gpurun_out/r2cfg; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 1800 python -m pytest tests/test_configs_gpu.py -q -k managed > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
