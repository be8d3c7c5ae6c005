#!/bin/bash
# Quick health pass: build, smoke, GPU parity tests, one default bench line.
R=gpurun_out/${1:-verify}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $R/smoke.log 2>&1; echo "rc=$?" >> $R/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > $R/pytest_gpu.log 2>&1; echo "rc=$?" >> $R/pytest_gpu.log
timeout 900 python bench.py > $R/bench_default.json 2> $R/bench_default.err
