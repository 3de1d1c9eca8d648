#!/bin/bash
# One-off box discovery: topology, host, PCIe DMA bandwidth.
out=gpurun_out/discovery
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
nvidia-smi topo -m > $out/topo.txt 2>&1
nvidia-smi -q > $out/smi_q.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
nproc > $out/nproc.txt
python -c 'import os; print(len(os.sched_getaffinity(0)))' > $out/affinity.txt
cat /proc/meminfo | head -5 > $out/meminfo.txt
ls /sys/class/iommu > $out/iommu.txt 2>&1
for d in /sys/bus/pci/devices/*; do if [ -f $d/class ] && grep -q 0x0302 $d/class; then echo "$d numa=$(cat $d/numa_node) speed=$(cat $d/current_link_speed) width=$(cat $d/current_link_width)"; fi; done > $out/gpu_pci.txt 2>&1
ls /sys/devices/system/node/ > $out/numa_nodes.txt 2>&1
cat /sys/kernel/mm/transparent_hugepage/enabled > $out/thp.txt 2>&1
python - > $out/h2d.txt 2>&1 <<'PY'
import torch, time
torch.cuda.init()
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for sz in [1<<20, 2<<20, 8<<20, 64<<20, 256<<20, 1<<30]:
    h = torch.empty(sz, dtype=torch.uint8).pin_memory()
    d = torch.empty(sz, dtype=torch.uint8, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    n = 10
    s.record()
    for _ in range(n): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)/n
    print(f"H2D {sz>>20} MiB: {sz/ms/1e6:.2f} GB/s ({ms:.3f} ms)")
    s.record()
    for _ in range(n): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)/n
    print(f"D2H {sz>>20} MiB: {sz/ms/1e6:.2f} GB/s")
PY
