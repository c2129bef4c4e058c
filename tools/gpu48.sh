#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p48_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p48_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p48_bench.json 2>&1
