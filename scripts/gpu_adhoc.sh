R=gpurun_out/hugetlb; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $R/build.log 2>&1
cat /proc/meminfo | grep -i huge > $R/meminfo.txt; free -g >> $R/meminfo.txt
timeout 900 python scripts/hugetlb_probe.py > $R/probe.jsonl 2> $R/probe.err
