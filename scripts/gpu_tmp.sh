R=gpurun_out/tests2; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $R/pytest_gpu.log 2>&1; echo rc=$? >> $R/pytest_gpu.log
