#!/bin/bash
for c in 16 24 96 148; do
CLO_GATHER_CTAS=$c timeout 1200 python bench.py --config 4 --batch 4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p59_c4_b4_c$c.json 2> /dev/null
done
