#!/bin/bash
# A/B: attention register cap, persistent flag-gated transfer kernel, gather CTAs; each twice.
run() { timeout 300 python bench.py --steps 32 --no-e2e --no-cpu-baseline > gpurun_out/p44_$1.json 2>&1; }
for rep in 1 2; do
run base_$rep
CLO_ATTN_REGCAP=255 run nocap_$rep
CLO_TRANSFER=flags run flags_$rep
CLO_GATHER_CTAS=96 run c96_$rep
done
