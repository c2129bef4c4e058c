# ncu launch list (durations) of configs[2]'s decode selection kernels
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:score|threshold|compact|reconcile|prepare|attn_mma|append|gather_engine' \
    --launch-skip 3000 --launch-count 200 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --config 3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_c2.log 2>&1
tail -2 gpurun_out/launches_c2.log
