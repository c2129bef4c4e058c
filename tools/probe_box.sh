#!/bin/bash
# One-off hardware probe of the GPU box (host RAM, CPU, PCIe topology, H2D bandwidth).
set -x
nvidia-smi
nvidia-smi topo -m
nvidia-smi -q | grep -iE -A3 "PCIe Generation|Link Width|Max Link"
free -g
nproc
lscpu | head -30
numactl -H 2>/dev/null || true
cat /proc/meminfo | head -5
ulimit -l
python - <<'PY'
import torch, time
x = torch.empty(1<<30, dtype=torch.uint8).pin_memory()
y = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
for i in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
best=0
for i in range(10):
    s.record(); y.copy_(x, non_blocking=True); e.record(); torch.cuda.synchronize()
    best=max(best, (1<<30)/(s.elapsed_time(e)*1e-3)/1e9)
print("H2D pinned GB/s best", best)
best=0
for i in range(10):
    s.record(); x.copy_(y, non_blocking=True); e.record(); torch.cuda.synchronize()
    best=max(best, (1<<30)/(s.elapsed_time(e)*1e-3)/1e9)
print("D2H pinned GB/s best", best)
print(torch.cuda.get_device_properties(0))
PY
