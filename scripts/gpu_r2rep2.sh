# round 2: --numa replica (pinned-thread fill) vs the default fill, alternating on one box
R=gpurun_out/r2rep2; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
for i in 1 2; do
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > $R/bench_default_$i.json 2> $R/bench_default_$i.err
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --numa replica > $R/bench_replica_$i.json 2> $R/bench_replica_$i.err
done
