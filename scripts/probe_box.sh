#!/bin/bash
# One-off box probe: topology, host RAM, NUMA, IOMMU, H2D memcpy ceiling.
set -x
nvidia-smi
nvidia-smi topo -m
free -g
nproc
lscpu | head -30
numactl -H 2>&1 | head -20
ls /sys/devices/system/node/
cat /proc/cmdline
cat /sys/kernel/mm/transparent_hugepage/enabled
cat /proc/meminfo | grep -i huge
ls /sys/kernel/iommu_groups | wc -l
dmesg 2>/dev/null | grep -i -E "iommu|dmar" | head
for d in /sys/bus/pci/devices/*; do if [ -f $d/class ] && grep -q 0x0302 $d/class; then echo $d $(cat $d/numa_node) $(cat $d/current_link_speed) $(cat $d/current_link_width); fi; done
python - <<'PY'
import torch, time
print(torch.cuda.get_device_properties(0))
p = torch.cuda.get_device_properties(0)
print("pci", p.pci_bus_id, p.pci_device_id, p.pci_domain_id)
n = 1<<30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
best=0
for i in range(10):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
    best=max(best, n/e0.elapsed_time(e1)/1e6)
print("H2D pinned 1GiB best GB/s", best)
best=0
for i in range(10):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
    best=max(best, n/e0.elapsed_time(e1)/1e6)
print("D2H pinned 1GiB best GB/s", best)
PY
