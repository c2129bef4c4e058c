#!/bin/bash
# MMA attention with cp.async staging: correctness, chunk sweep, ncu.
timeout 900 python -m pytest tests -m gpu -x -q -k "engine or edge or fullsize or ops" > gpurun_out/p24_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p24_tests.log
for ch in 256 512 768; do
CLO_ATTN_CHUNK=$ch timeout 300 python bench.py --steps 24 --no-e2e --no-cpu-baseline > gpurun_out/p24_bench_c$ch.json 2>&1
done
CLO_ATTN=tma timeout 300 python bench.py --steps 24 --no-e2e --no-cpu-baseline > gpurun_out/p24_bench_tma.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_mma" -s 40 -c 1 -o gpurun_out/p24_attn_mma -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p24_ncu.log 2>&1
