#!/bin/bash
# Flat (all-SM) vs head-aligned segments for the MMA attention.
for sh in 4x3x2x16 4x6x1x16 4x3x1x32 8x3x1x16; do
CLO_ATTN_ALIGN=0 CLO_ATTN_SHAPE=$sh timeout 300 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p32_bench_flat_$sh.json 2>&1
done
CLO_ATTN_ALIGN=0 CLO_ATTN_SHAPE=4x3x2x16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_mma" -s 80 -c 1 -o gpurun_out/p32_attn_mma -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p32_ncu.log 2>&1
