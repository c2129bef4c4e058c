#!/bin/bash
# Reproduces the profiles/ captures on a B200 box (run through gpurun from the repo root):
#   bash tools/evidence.sh
# Writes gpurun_out/ev_*; profiles/README.md summarises the numbers.
set -u
# default bench line (configs[1]) and every BASELINE config once
timeout 600 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
for c in 1 3 4; do
  timeout 1500 python bench.py --config $c --steps 8 --warmup 3 --no-e2e > gpurun_out/ev_config$c.json 2>/dev/null
done
# decode-step launch list (skip setup + prefill), serialised, cold caches
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# full captures of the attention and score kernels of a decode layer
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_mma_stream" -s 60 -c 1 \
  -o gpurun_out/ev_attn -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_signhash" -s 300 -c 1 \
  -o gpurun_out/ev_score -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# full capture of one engine gather launch (the first: a prefill layer, 128 heads x 2048 rows)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_engine" -c 1 \
  -o gpurun_out/ev_gather -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# zero-copy gather sweep (configs[4])
timeout 900 python bench_gather.py > gpurun_out/ev_gather_sweep.jsonl 2>&1
