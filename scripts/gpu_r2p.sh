# round 2 pass p: gather_multi test; ncu of the e2e direct-store kernel (upstream bytes)
R=gpurun_out/r2p; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 900 python -m pytest tests/test_round2_gpu.py -q -k "multi or gather_host" > $R/pytest.log 2>&1; echo "rc=$?" >> $R/pytest.log
TM=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sectors_aperture_sysmem_op_read.sum,syslts__t_requests_aperture_sysmem_op_read.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__read_bytes.sum.per_second,pcie__write_bytes.sum.per_second
timeout 1200 ncu --nvtx --nvtx-include e2e/ -k regex:'k_(single|multi)' --metrics $TM --clock-control none --csv --log-file $R/e2e_papers.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-check --max-lists 7 > $R/e2e_papers.json 2> $R/e2e_papers.err
