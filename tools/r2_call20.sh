set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c20_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
CLO_BENCH_SPANS=gpurun_out/r2_c20_spans_c128.json $B > gpurun_out/r2_c20_c128.json 2>&1
CLO_SELECT_CLUSTER=4 CLO_BENCH_SPANS=gpurun_out/r2_c20_spans_cl4.json $B > gpurun_out/r2_c20_cl4.json 2>&1
CLO_GATHER_CTAS=64 CLO_BENCH_SPANS=gpurun_out/r2_c20_spans_c64.json $B > gpurun_out/r2_c20_c64.json 2>&1
