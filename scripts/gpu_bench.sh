#!/bin/bash
# Bench runs + launch list + one full ncu capture of the gather kernel. Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in products reddit; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --config sweep:512 --no-cpu --no-e2e > gpurun_out/bench_sweep512.json 2> gpurun_out/bench_sweep512.err
timeout 600 python bench.py --config sweep:512 --no-cpu --no-e2e --plan reorder=off > gpurun_out/bench_sweep512_noreorder.json 2>> gpurun_out/bench_sweep512.err
timeout 600 python bench.py --impl reference --steps 10 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_products.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 4 -c 1 -o gpurun_out/prof_products python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --max-lists 6 > gpurun_out/ncu_full.log 2>&1
