#!/bin/bash
# quick_bw for every variant in build/variants (1-GiB table, inside the translation reach)
mkdir -p gpurun_out
for so in build/variants/libut_*.so; do
  n=$(basename $so .so)
  echo "== $n" >> gpurun_out/variants.log
  UT_LIB=$so timeout 300 python scripts/quick_bw.py --table-gib 1 --widths "$@" >> gpurun_out/variants.log 2>&1
done
