# ncu --set full of one decode-layer attention launch at configs[2] (bench --config 3)
ncu --set full --clock-control none --import-source on -k regex:attn_mma_stream --launch-skip 150 --launch-count 1 \
    -o gpurun_out/ncu_attn_c2 -f python bench.py --config 3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_attn_c2.log 2>&1
ncu -i gpurun_out/ncu_attn_c2.ncu-rep --page details --csv > gpurun_out/ncu_attn_c2_details.csv 2>&1
tail -3 gpurun_out/ncu_attn_c2.log
