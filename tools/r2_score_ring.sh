# 4-stage score ring: GPU tests, configs[1]/[2] bench, decode launch list at configs[1]
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests5.log 2>&1; tail -3 gpurun_out/gputests5.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ring_c2.json 2> gpurun_out/ring_c2.err
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/ring_c3.json 2> gpurun_out/ring_c3.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv \
  --log-file gpurun_out/ring_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
