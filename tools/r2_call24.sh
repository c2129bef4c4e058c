set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c24_gputest.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B --steps 30 > gpurun_out/r2_c24_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_signhash" -s 300 -c 1 -o gpurun_out/r2_ncu_score2 -f $B --steps 2 --warmup 3 > /dev/null 2>&1
