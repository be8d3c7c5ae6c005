# round 2, last session: pool tables from four threads at once (shared slab / scratch pool), the C
# example on both GPU backends, smoke with the recycled pool table
R=gpurun_out/r2pool3; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 900 python -m pytest tests/test_pool.py tests/test_c_example.py tests/test_unified_api.py -q -m gpu > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
