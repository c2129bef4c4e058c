#!/bin/bash
# Batched combine: tests + aligned/flat shape sweep.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p34_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p34_tests.log
for sh in 8x3x1x16 4x6x1x16 4x3x1x32; do
CLO_ATTN_SHAPE=$sh timeout 300 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p34_bench_al_$sh.json 2>&1
CLO_ATTN_ALIGN=0 CLO_ATTN_SHAPE=$sh timeout 300 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p34_bench_flat_$sh.json 2>&1
done
CLO_ATTN_ALIGN=0 CLO_ATTN_SHAPE=4x3x2x16 timeout 300 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p34_bench_flat_4x3x2x16.json 2>&1
