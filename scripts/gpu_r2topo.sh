# round 2: host-link facts in the bench line (PCIe gen/width, GPU pairs)
R=gpurun_out/r2topo; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
nvidia-smi topo -m > $R/topo.txt 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "box_harness_tiny or two_workers_one_gpu" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $R/bench_default.json 2> $R/bench_default.err
