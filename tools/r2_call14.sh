set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c14_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
CLO_BENCH_SPANS=gpurun_out/r2_c14_spans_c128.json $B > gpurun_out/r2_c14_c128.json 2>&1
CLO_SELECT_CLUSTER=8 CLO_BENCH_SPANS=gpurun_out/r2_c14_spans_cl8.json $B > gpurun_out/r2_c14_cl8.json 2>&1
CLO_GATHER_CTAS=48 CLO_BENCH_SPANS=gpurun_out/r2_c14_spans_c48.json $B > gpurun_out/r2_c14_c48.json 2>&1
