# compact_quota for 512K items (129 chunks): configs[2] A/B, alternating
for i in 1 2; do
  CLO_QUOTA_MAX_CHUNKS=160 timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/ql_on_$i.json
  timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/ql_off_$i.json
done
CLO_QUOTA_MAX_CHUNKS=160 timeout 900 python -m pytest tests/test_gpu_longctx.py -q -x > gpurun_out/ql_tests.log 2>&1; tail -1 gpurun_out/ql_tests.log
