set -u
CLO_GATHER=wide_smem timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_edge_cases.py tests/test_gpu_transfer_modes.py -x -q > gpurun_out/r2_c35_test.log 2>&1
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 30"
$B > gpurun_out/r2_c35_def.json 2>&1
for c in 12 16 20; do CLO_GATHER=wide_smem CLO_GATHER_CTAS=$c CLO_BENCH_SPANS=gpurun_out/r2_c35_spans_$c.json $B > gpurun_out/r2_c35_ws$c.json 2>&1; done
CLO_GATHER=wide_smem CLO_GATHER_CTAS=16 CLO_GATHER_WIDE=1 $B > gpurun_out/r2_c35_ws16_s1.json 2>&1
CLO_GATHER=wide_smem CLO_GATHER_CTAS=16 CLO_GATHER_WIDE=3 $B > gpurun_out/r2_c35_ws16_s3.json 2>&1
$B > gpurun_out/r2_c35_def2.json 2>&1
