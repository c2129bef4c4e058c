#!/bin/bash
# Unrolled FP64 chains: correctness + ncu of prepare/append + bench.
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p41_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p41_tests.log
timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p41_bench.json 2>&1
CLO_BENCH_SPANS=gpurun_out/p41_spans.json timeout 300 python bench.py --steps 8 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"prepare_kernel|append_kernel" -s 200 -c 4 -o gpurun_out/p41_sel -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p41_ncu.log 2>&1
