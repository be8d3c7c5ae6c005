R=gpurun_out/tma4; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 300 python scripts/quick_bw.py --table-gib 0.9 --widths 16,64,128,256,400,512,1024 --plans auto,bulk,tma4 > $R/bw.jsonl 2> $R/bw.err
timeout 900 python -m pytest tests/test_gather_gpu.py -q -x -k "randomized or guard" > $R/pytest.log 2>&1; echo rc=$? >> $R/pytest.log
timeout 900 python -m pytest tests/test_sanitizer_gpu.py -q -x > $R/sanitize.log 2>&1; echo rc=$? >> $R/sanitize.log
