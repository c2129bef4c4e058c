#!/bin/bash
# Step-level A/B: attention smem footprint vs co-scheduling of the selection chain; selection priority.
run() { timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p38_$1.json 2>&1; }
CLO_ATTN_SHAPE=8x3x1x16 run a8x3
CLO_ATTN_SHAPE=4x3x1x32 run a4x3x32
CLO_ATTN_SHAPE=4x3x2x16 CLO_ATTN_ALIGN=1 run a4x3x2
CLO_ATTN=tma run tma
CLO_SEL_PRIO=high CLO_ATTN_SHAPE=8x3x1x16 run a8x3_selhi
CLO_SEL_PRIO=high CLO_ATTN_SHAPE=4x3x1x32 run a4x3x32_selhi
