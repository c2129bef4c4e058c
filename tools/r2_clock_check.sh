# clock sampler started before the warm-up: default line, configs[0] long enough for samples, GPU contract tests
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ck_c2.json 2> gpurun_out/ck_c2.err
timeout 600 python bench.py --config 1 --steps 200 --warmup 5 > gpurun_out/ck_c1.json 2> gpurun_out/ck_c1.err
timeout 600 python bench.py --config 1 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ck_c1_short.json 2>/dev/null
timeout 600 python -m pytest tests/test_bench_contract.py -q > gpurun_out/ck_contract.log 2>&1; tail -1 gpurun_out/ck_contract.log
