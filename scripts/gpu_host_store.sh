# round 2: TMA bulk stores vs 16-B SM stores into mapped host memory (PCIe write bytes)
R=gpurun_out/hst; mkdir -p $R
timeout 300 build/probes/host_store_probe > $R/host_store.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__write_bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum.per_second --clock-control none --csv --log-file $R/host_store_ncu.csv build/probes/host_store_probe > $R/host_store_under_ncu.jsonl 2>&1
