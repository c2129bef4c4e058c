#!/bin/bash
# Box probe + PCIe gather payload efficiency vs row width + bench variance vs gather CTAs.
nvidia-smi topo -m > gpurun_out/p21_topo.txt 2>&1
(lscpu; numactl -H; cat /proc/meminfo | head -3; cat /sys/class/pci_bus/*/device/numa_node 2>/dev/null | sort | uniq -c) > gpurun_out/p21_host.txt 2>&1
nvidia-smi -q | grep -iE -A2 "Bus Id|PCIe Generation|Link Width" >> gpurun_out/p21_host.txt
timeout 300 python bench_gather.py --d 128 --rows 2048,8192 --skip-cpu > gpurun_out/p21_gather_d128.jsonl 2>&1
timeout 300 python bench_gather.py --d 256 --rows 1024,4096 --skip-cpu > gpurun_out/p21_gather_d256.jsonl 2>&1
timeout 300 python bench_gather.py --d 128 --rows 2048,8192 --skip-cpu --huge > gpurun_out/p21_gather_d128_huge.jsonl 2>&1
for c in 48 96 148; do
  CLO_GATHER_CTAS=$c timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p21_bench_c$c.json 2>&1
done
timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p21_bench_again.json 2>&1
