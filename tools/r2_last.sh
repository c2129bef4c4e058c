# last-tree bench line, reference arm, smoke, decode launch list
timeout 600 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/last_ref.json 2> /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; tail -1 gpurun_out/last_smoke.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv \
  --log-file gpurun_out/last_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
