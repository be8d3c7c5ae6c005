# round 2 pass d: order experiments on the 16-GiB managed sweep table (partial-line widths)
R=gpurun_out/r2d; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
for rb in 400 516 260 2052 128 64; do
  for v in "" "--plan reorder=on" "--presort"; do
    echo "== rb=$rb $v" >> $R/sweep_order.log
    timeout 600 python bench.py --config sweep:$rb --steps 10 --warmup 3 --no-cpu --no-e2e --max-lists 13 $v >> $R/sweep_order.log 2>&1
  done
done
