# round 2 pass q: new harness tests
R=gpurun_out/r2q; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 1800 python -m pytest tests/test_round2_gpu.py -q > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
