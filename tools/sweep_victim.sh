#!/bin/bash
# victim-row pool size sweep at configs[1] (tokens/s vs PCIe bytes)
for v in ${VICTIMS:-0 2048 4096 8192 16384}; do
  timeout 600 python bench.py --steps 30 --no-e2e --no-cpu-baseline --victim-rows $v > gpurun_out/r2_victim_$v.json 2> gpurun_out/r2_victim_$v.err
done
