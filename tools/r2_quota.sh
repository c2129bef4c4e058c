# threshold folded into compaction (per-CTA quota): GPU tests, A/B on configs[1], configs[0], launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests8.log 2>&1; tail -1 gpurun_out/gputests8.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_on_a.json 2> gpurun_out/q_on_a.err
CLO_COMPACT_QUOTA=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_off.json 2> /dev/null
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_on_b.json 2> /dev/null
timeout 600 python bench.py --config 1 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/q_c1.json 2> /dev/null
CLO_BENCH_SPANS=gpurun_out/spans_quota.json timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 8 > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1000 -c 700 --csv \
  --log-file gpurun_out/q_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
