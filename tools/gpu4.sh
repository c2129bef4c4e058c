set -x
timeout 900 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-1500
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 900 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prepare|threshold|reconcile|compact|score_signhash" -s 50 -c 10 -o gpurun_out/prof_sel -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_sel.log 2>&1
