# Harley-Seal popcount in the score kernel: GPU tests, configs[1] x2, configs[2], launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests7.log 2>&1; tail -1 gpurun_out/gputests7.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/popc_c2a.json 2> gpurun_out/popc_c2a.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/popc_c2b.json 2> /dev/null
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/popc_c3.json 2> /dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv \
  --log-file gpurun_out/popc_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
