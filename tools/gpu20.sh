timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q 2>&1 | tail -15
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_tma" -s 40 -c 2 -o gpurun_out/prof_attn3 -f python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn3.log 2>&1
tail -1 gpurun_out/ncu_attn3.log
