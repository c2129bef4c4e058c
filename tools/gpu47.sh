#!/bin/bash
# Decode-step launch list (skip setup + prefill) and full captures of loaded gather / score launches.
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv --log-file gpurun_out/p47_launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p47_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_engine" -s 300 -c 1 -o gpurun_out/p47_gather -f \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_signhash" -s 300 -c 1 -o gpurun_out/p47_score -f \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
