# round 2 pass g: in-process coop on one device — which environment is needed
R=gpurun_out/r2g; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
for w in 2 3; do
  echo "== w=$w both" >> $R/coop_local.log
  CUDA_MODULE_LOADING=EAGER CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 150 python tests/coop_local_case.py $w >> $R/coop_local.log 2>&1; echo "rc=$?" >> $R/coop_local.log
  echo "== w=$w maxconn only" >> $R/coop_local.log
  CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 120 python tests/coop_local_case.py $w >> $R/coop_local.log 2>&1; echo "rc=$?" >> $R/coop_local.log
  echo "== w=$w eager only" >> $R/coop_local.log
  CUDA_MODULE_LOADING=EAGER timeout 150 python tests/coop_local_case.py $w >> $R/coop_local.log 2>&1; echo "rc=$?" >> $R/coop_local.log
  echo "== w=$w neither" >> $R/coop_local.log
  timeout 120 python tests/coop_local_case.py $w >> $R/coop_local.log 2>&1; echo "rc=$?" >> $R/coop_local.log
done
timeout 300 python bench.py --gpus 2 --oversubscribe --coop device --config products --steps 20 --warmup 5 --no-cpu > $R/box2_products_coop.json 2> $R/box2_products_coop.err; echo "rc=$?" >> $R/box2_products_coop.err
timeout 300 python bench.py --gpus 4 --oversubscribe --coop device --config reddit --steps 20 --warmup 5 --no-cpu > $R/box4_reddit_coop.json 2> $R/box4_reddit_coop.err; echo "rc=$?" >> $R/box4_reddit_coop.err
timeout 300 python bench.py --gpus 4 --oversubscribe --config reddit --steps 20 --warmup 5 --no-cpu --no-e2e > $R/box4_reddit.json 2> $R/box4_reddit.err; echo "rc=$?" >> $R/box4_reddit.err
