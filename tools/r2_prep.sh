# prepare: one-round-trip staging + early P-slice copy: GPU tests, configs[1] x2, configs[2], launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests6.log 2>&1; tail -1 gpurun_out/gputests6.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/prep_c2a.json 2> gpurun_out/prep_c2a.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/prep_c2b.json 2> /dev/null
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/prep_c3.json 2> /dev/null
CLO_BENCH_SPANS=gpurun_out/spans_prep.json timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 8 > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv \
  --log-file gpurun_out/prep_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
