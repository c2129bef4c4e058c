set -u
CLO_GATHER=wide timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_edge_cases.py tests/test_gpu_transfer_modes.py -x -q > gpurun_out/r2_c34_widetest.log 2>&1
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 30"
$B > gpurun_out/r2_c34_def.json 2>&1
for c in 16 20 24; do CLO_GATHER=wide CLO_GATHER_CTAS=$c CLO_BENCH_SPANS=gpurun_out/r2_c34_spans_w$c.json $B > gpurun_out/r2_c34_wide$c.json 2>&1; done
CLO_GATHER=wide CLO_GATHER_CTAS=20 CLO_GATHER_RESERVE=0 $B > gpurun_out/r2_c34_wide20_nores.json 2>&1
CLO_GATHER=wide CLO_GATHER_CTAS=20 CLO_GATHER_WIDE=3 $B > gpurun_out/r2_c34_wide20_1024.json 2>&1
CLO_GATHER=wide CLO_GATHER_CTAS=20 CLO_GATHER_WIDE=1 $B > gpurun_out/r2_c34_wide20_u8.json 2>&1
