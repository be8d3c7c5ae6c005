# round 2, last session: the recycling unified allocator (ut_pool_*) on the GPU — its tests, the
# unified-tensor tests, and what recycling saves per tensor (scripts/pool_probe.py)
R=gpurun_out/r2pool; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_pool.py tests/test_unified_api.py tests/test_abi.py -q -m "gpu or not gpu" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python scripts/pool_probe.py > $R/pool_probe.jsonl 2> $R/pool_probe.err
