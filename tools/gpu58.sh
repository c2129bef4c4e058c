#!/bin/bash
for b in 1 2 4; do
timeout 1200 python bench.py --config 4 --batch $b --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p58_c4_b$b.json 2> gpurun_out/p58_c4_b$b.err
done
timeout 1200 python bench.py --config 2 --ctx 524288 --batch 4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p58_c2_512k_b4.json 2> gpurun_out/p58_c2.err
