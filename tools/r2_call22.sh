set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c22_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 30"
CLO_BENCH_SPANS=gpurun_out/r2_c22_spans_c128.json $B > gpurun_out/r2_c22_c128.json 2>&1
CLO_CHAIN_SELECT=0 CLO_BENCH_SPANS=gpurun_out/r2_c22_spans_unchained.json $B > gpurun_out/r2_c22_unchained.json 2>&1
CLO_GATHER_CTAS=64 CLO_BENCH_SPANS=gpurun_out/r2_c22_spans_c64.json $B > gpurun_out/r2_c22_c64.json 2>&1
