set -u
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
for c in 16 32 64; do CLO_GATHER_CTAS=$c CLO_BENCH_SPANS=gpurun_out/r2_spans_c$c.json $B > gpurun_out/r2_ctas_$c.json 2>&1; done
CLO_GATHER_CTAS=32 CLO_GATHER_TMA_SHAPE=1,2 CLO_BENCH_SPANS=gpurun_out/r2_spans_c32s2.json $B > gpurun_out/r2_ctas_32s2.json 2>&1
CLO_GATHER=lsu CLO_GATHER_CTAS=16 CLO_BENCH_SPANS=gpurun_out/r2_spans_lsu16.json $B > gpurun_out/r2_ctas_lsu16.json 2>&1
