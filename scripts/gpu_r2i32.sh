# round 2: ut_gather_i32 (parity tests + sanitizer over every case incl. int32 ids)
R=gpurun_out/r2i32; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py tests/test_sanitizer_gpu.py -q > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
