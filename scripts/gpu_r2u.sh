R=gpurun_out/r2u; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "sampling" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
