#!/bin/bash
# Gather CTA count re-tune with the tensor-core attention in the step.
for c in 48 72 96 128 148; do
CLO_GATHER_CTAS=$c timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p35_bench_c$c.json 2>&1
done
