#!/bin/bash
# Neighbour line sharing: parity tests, then products A/B (share off vs on).
R=gpurun_out/${1:-share}
mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_gather_gpu.py -q -m gpu -k "share or randomized or guard" > $R/pytest_share.log 2>&1; echo "rc=$?" >> $R/pytest_share.log
for i in 1 2 3; do
  for m in off on; do
    timeout 600 python bench.py --plan share=$m --steps 50 --no-cpu --no-e2e >> $R/bench_products_share_$m.jsonl 2>> $R/bench.err
  done
done
for m in off on; do
  timeout 600 python bench.py --config reddit --plan share=$m --steps 30 --no-cpu --no-e2e >> $R/bench_reddit_share_$m.jsonl 2>> $R/bench.err
done
TM=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sectors_aperture_sysmem_op_read.sum,syslts__t_requests_aperture_sysmem_op_read.sum,pcie__read_bytes.sum
for m in off on; do
  timeout 600 ncu --nvtx --nvtx-include timed/ -k regex:'k_(single|share)' --metrics $TM --clock-control none --csv --log-file $R/traffic_products_share_$m.csv python bench.py --plan share=$m --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > /dev/null 2>&1
done
