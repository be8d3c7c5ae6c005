# the load kernel alone after the k_req-like index load
R=gpurun_out/r2ll; mkdir -p $R
timeout 300 build/probes/loaded_latency_probe 4 22 1 0 > $R/load_only_fixed.jsonl 2>&1
