# round 2 pass v: order strategies on the papers-shaped REGISTERED table (translation-bound memory)
R=gpurun_out/r2v; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
B="python bench.py --config papers --alloc register --steps 20 --warmup 5 --no-cpu --no-e2e"
for v in "" "--plan exact=on" "--plan exact=on,conc=dense" "--plan conc=dense" "--presort --plan reorder=off" "--presort --plan reorder=off,conc=sparse"; do
  echo "== $v" >> $R/papers_registered_order.log
  timeout 900 $B $v >> $R/papers_registered_order.log 2>&1
done
echo "== managed exact" >> $R/papers_registered_order.log
timeout 900 python bench.py --config papers --steps 20 --warmup 5 --no-cpu --no-e2e --plan reorder=on,exact=on >> $R/papers_registered_order.log 2>&1
