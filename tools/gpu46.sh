#!/bin/bash
# Round-1 evidence: launch list of the default bench (serialised, cold), ncu --set full of the
# attention kernel and of one decode-step gather, and the default bench line.
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/p46_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p46_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_mma_stream" -s 60 -c 1 -o gpurun_out/p46_attn -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_engine" -s 40 -c 1 -o gpurun_out/p46_gather -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_signhash" -s 60 -c 1 -o gpurun_out/p46_score -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/p46_bench.json 2> gpurun_out/p46_bench.err
