R=gpurun_out/coop1; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_coop_gpu.py -v -x --timeout 300 -k "world1 or bad" > $R/pytest_w1.log 2>&1; echo rc=$? >> $R/pytest_w1.log
timeout 900 python -m pytest tests/test_coop_gpu.py -v -x --timeout 300 -k "processes" > $R/pytest_mp.log 2>&1; echo rc=$? >> $R/pytest_mp.log
