#!/bin/bash
# ncu evidence only (the tail of gpu_round.sh): launch lists, per-launch traffic, one full capture
# per workload, all restricted to bench.py's NVTX "timed" range. Usage: gpu_ncu.sh DIR [configs...]
R=gpurun_out/${1:-ncu}; shift
mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
NV='--nvtx --nvtx-include timed/'
TM=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sectors_aperture_sysmem_op_read.sum,syslts__t_requests_aperture_sysmem_op_read.sum,pcie__read_bytes.sum
for c in ${@:-products}; do
  timeout 900 ncu $NV --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches_$c.csv python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > /dev/null 2>&1
  timeout 900 ncu $NV -k regex:'k_(single|multi|narrow|runs)' --metrics $TM --clock-control none --csv --log-file $R/traffic_$c.csv python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > $R/traffic_$c.json 2> $R/traffic_$c.err
  timeout 900 ncu $NV -k regex:'k_single|k_multi' -s 2 -c 1 --set full --clock-control none --import-source on -o $R/prof_$c python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > $R/ncu_full_$c.log 2>&1
done
