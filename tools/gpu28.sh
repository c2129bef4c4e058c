#!/bin/bash
# MMA attention shapes A/B + tests + ncu of the default shape.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p28_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p28_tests.log
for sh in 4x6x1 4x3x2 8x3x1; do
CLO_ATTN_SHAPE=$sh timeout 300 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p28_bench_$sh.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_mma" -s 80 -c 2 -o gpurun_out/p28_attn_mma -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p28_ncu.log 2>&1
