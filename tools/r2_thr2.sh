# packed-register threshold: select/engine GPU tests, configs[2]/[1] bench, threshold launch durations at configs[2]
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests4.log 2>&1; tail -3 gpurun_out/gputests4.log
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/thr2_c3.json 2> gpurun_out/thr2_c3.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/thr2_c2.json 2> gpurun_out/thr2_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:threshold|score_signhash|compact|reconcile' \
    --launch-skip 400 --launch-count 60 --csv --log-file gpurun_out/launches_thr2_c2.csv \
    python bench.py --config 3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
