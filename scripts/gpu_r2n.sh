# round 2 pass n: ncu for reddit on the managed table (roofline.traffic of every graphsage config)
R=gpurun_out/r2n; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
NV='--nvtx --nvtx-include timed/'
TM=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sectors_aperture_sysmem_op_read.sum,syslts__t_requests_aperture_sysmem_op_read.sum,pcie__read_bytes.sum,pcie__write_bytes.sum
for c in reddit; do
  timeout 900 ncu $NV --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches_$c.csv python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > $R/launches_$c.json 2>&1
  timeout 900 ncu $NV -k regex:'k_(single|multi|narrow|runs|share)' --metrics $TM --clock-control none --csv --log-file $R/traffic_$c.csv python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > $R/traffic_$c.json 2> $R/traffic_$c.err
  timeout 900 ncu $NV -k regex:'k_single|k_multi|k_share[^_]|k_share$' -s 2 -c 1 --set full --clock-control none --import-source on -o $R/prof_$c python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > $R/ncu_full_$c.log 2>&1
done
