#!/bin/bash
# Build, smoke, GPU parity tests, quick bandwidth probe. Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/quick_bw.py "$@" > gpurun_out/quick_bw.log 2>&1; echo "bw rc=$?" >> gpurun_out/quick_bw.log
