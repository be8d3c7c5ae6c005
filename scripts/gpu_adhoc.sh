R=gpurun_out/misc3; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
timeout 300 python scripts/e2e_pipe_probe.py products > $R/pipe.jsonl 2> $R/pipe.err
timeout 300 python bench.py --config sweep:64 --steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13 > $R/sweep64.json 2> $R/sweep64.err
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches_coop_products.csv python bench.py --coop device --steps 6 --warmup 3 --no-e2e --no-cpu --max-lists 9 > $R/coop_ncu.json 2> $R/coop_ncu.err
