set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 900 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-2500
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_tma|append" -s 40 -c 4 -o gpurun_out/prof_attn2 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn2.log 2>&1
