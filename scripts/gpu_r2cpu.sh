# round 2: the CPU-centric baseline's spread within one lease (host model/L3 recorded)
R=gpurun_out/r2cpu; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
lscpu > $R/lscpu.txt 2>&1
for i in 1 2 3; do
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e > $R/bench_default_$i.json 2> $R/bench_default_$i.err
done
