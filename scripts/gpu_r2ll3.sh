# round 2: reads beside host stores (the host->host gather's two directions), loaded latency
R=gpurun_out/r2ll; mkdir -p $R
timeout 600 build/probes/loaded_latency_probe 4 22 0 2 1 > $R/duplex.jsonl 2>&1
