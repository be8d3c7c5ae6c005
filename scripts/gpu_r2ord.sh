# round 2: does visiting order matter for the managed papers-shaped table (512-B whole-line rows)?
R=gpurun_out/r2ord; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
for v in "" "--plan reorder=on" "--presort" "--plan reorder=on,exact=on"; do
  echo "== $v" >> $R/order.log
  timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --no-e2e $v >> $R/order.log 2>> $R/order.err
done
