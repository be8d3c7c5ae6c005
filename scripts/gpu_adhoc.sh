R=gpurun_out/cooprand; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_coop_gpu.py -q -x --timeout 300 -k "randomized or world1" > $R/pytest.log 2>&1; echo rc=$? >> $R/pytest.log
