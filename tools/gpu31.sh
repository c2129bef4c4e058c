#!/bin/bash
# MMA attention tile/shape sweep + tests + ncu of the default.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p31_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p31_tests.log
for sh in 4x3x1x32 8x2x1x32 8x3x1x16 4x6x1x16; do
CLO_ATTN_SHAPE=$sh timeout 300 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p31_bench_$sh.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_mma" -s 80 -c 1 -o gpurun_out/p31_attn_mma -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p31_ncu.log 2>&1
