# round 2: request-rate probe + ncu request/PCIe counters + calibration (VERDICT r1 task 4)
R=gpurun_out/${1:-req1}; mkdir -p $R
P=build/probes/request_rate_probe
timeout 600 $P 4 managed > $R/request_rate_managed.jsonl 2>&1
timeout 600 $P 1 pinned > $R/request_rate_pinned.jsonl 2>&1
TM=gpu__time_duration.sum,syslts__t_requests_aperture_sysmem_op_read.sum,syslts__t_sectors_aperture_sysmem_op_read.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $TM --clock-control none --csv --log-file $R/request_rate_ncu.csv $P 4 managed > $R/request_rate_under_ncu.jsonl 2>&1
