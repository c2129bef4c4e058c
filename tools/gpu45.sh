#!/bin/bash
run() { timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p45_$1.json 2>&1; }
for rep in 1 2; do
run base_$rep
CLO_TRANSFER=flags run flags_$rep
CLO_GATHER_CTAS=64 run c64_$rep
CLO_GATHER_CTAS=32 run c32_$rep
CLO_TRANSFER=flags CLO_GATHER_CTAS=64 run flags64_$rep
done
