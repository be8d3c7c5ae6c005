#!/bin/bash
mkdir -p gpurun_out
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_requests_aperture_sysmem_op_read.sum,syslts__t_sectors_aperture_sysmem_op_read.sum,syslts__d_sectors_fill_sysmem.sum,syslts__t_requests_aperture_sysmem_op_read_lookup_miss.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_read.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_cases.csv python scripts/ncu_cases.py > gpurun_out/ncu_cases.log 2>&1
