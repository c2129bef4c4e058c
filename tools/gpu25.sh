#!/bin/bash
# Persistent MMA attention: correctness, bench A/B, ncu.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p25_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p25_tests.log
timeout 300 python bench.py --steps 24 --no-e2e --no-cpu-baseline > gpurun_out/p25_bench_mma.json 2>&1
CLO_ATTN=tma timeout 300 python bench.py --steps 24 --no-e2e --no-cpu-baseline > gpurun_out/p25_bench_tma.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_mma" -s 80 -c 2 -o gpurun_out/p25_attn_mma -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p25_ncu.log 2>&1
