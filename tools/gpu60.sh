#!/bin/bash
CLO_GATHER=tma timeout 1200 python -m pytest tests -m gpu -x -q -k "engine or edge or fullsize or trace" > gpurun_out/p60_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p60_tests.log
CLO_GATHER=tma timeout 600 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p60_c2_tma.json 2>/dev/null
timeout 600 python bench.py --steps 16 --no-e2e --no-cpu-baseline > gpurun_out/p60_c2_lsu.json 2>/dev/null
CLO_GATHER=tma timeout 1200 python bench.py --config 4 --batch 4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p60_c4_tma.json 2>/dev/null
timeout 1200 python bench.py --config 4 --batch 4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p60_c4_lsu.json 2>/dev/null
