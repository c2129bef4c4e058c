#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p43_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p43_tests.log
timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p43_bench.json 2>&1
CLO_BENCH_SPANS=gpurun_out/p43_spans.json timeout 300 python bench.py --steps 8 --no-e2e --no-cpu-baseline > /dev/null 2>&1
