# round 2: whole-list error positions from chunked gathers (reorder > 2^31 rows, ut_gather_host pipeline)
R=gpurun_out/r2pos; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 1500 python -m pytest tests/test_round2_gpu.py tests/test_gather_gpu.py -q -k "beyond_2pow31 or error_position or gather_host or out_of_range or guard" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python -m pytest tests/test_sanitizer_gpu.py -q > $R/sanitizer.log 2>&1; echo "rc=$?" >> $R/sanitizer.log
