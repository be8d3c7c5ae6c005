R=gpurun_out/r2z; mkdir -p $R
python scripts/probes/hostnuma_advise_probe.py > $R/hostnuma_probe.jsonl 2>&1
ls /sys/devices/system/node/ >> $R/hostnuma_probe.jsonl 2>&1
cat /proc/cmdline >> $R/hostnuma_probe.jsonl 2>&1
