set -u
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv --log-file gpurun_out/r2_launches.csv $B --steps 4 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_signhash" -s 300 -c 1 -o gpurun_out/r2_ncu_score -f $B --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reconcile_kernel" -s 60 -c 1 -o gpurun_out/r2_ncu_reconcile -f $B --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prepare_kernel" -s 60 -c 1 -o gpurun_out/r2_ncu_prepare -f $B --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_mma_stream" -s 60 -c 1 -o gpurun_out/r2_ncu_attn -f $B --steps 2 --warmup 3 > /dev/null 2>&1
