# round 2: loaded latency x request rate (Little's law) on the managed host table
R=gpurun_out/r2ll; mkdir -p $R
timeout 600 build/probes/loaded_latency_probe 4 22 > $R/loaded_latency.jsonl 2>&1
