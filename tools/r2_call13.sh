set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c13_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
for c in 128 48; do CLO_GATHER_CTAS=$c CLO_BENCH_SPANS=gpurun_out/r2_c13_spans_c$c.json $B > gpurun_out/r2_c13_ctas_$c.json 2>&1; done
CLO_FUSED_SELECT=0 CLO_BENCH_SPANS=gpurun_out/r2_c13_spans_unfused.json $B > gpurun_out/r2_c13_unfused.json 2>&1
