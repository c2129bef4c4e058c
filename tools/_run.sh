#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p62_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p62_tests.log
timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p62_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_mma_stream" -s 60 -c 1 -o gpurun_out/p62_attn -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
