timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prepare_kernel|append_kernel" -s 70 -c 4 -o gpurun_out/prof_pa -f python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pa.log 2>&1
tail -2 gpurun_out/ncu_pa.log
