#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p52_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p52_tests.log
timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p52_bench_tma.json 2>&1
CLO_SCORE=lsu timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p52_bench_lsu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_signhash" -s 300 -c 1 -o gpurun_out/p52_score -f \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
