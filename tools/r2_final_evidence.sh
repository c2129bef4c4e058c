#!/bin/bash
# Round-2 closing evidence (run through gpurun from the repo root): default bench line,
# reference arm, every BASELINE config, decode launch list, ncu --set full of the
# attention / score / threshold kernels (details exported as CSV on the box).
set -u
timeout 600 python bench.py > gpurun_out/ev2_bench.json 2> gpurun_out/ev2_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/ev2_ref.json 2> gpurun_out/ev2_ref.err
for c in 1 3 4; do
  timeout 1500 python bench.py --config $c --steps 8 --warmup 3 --no-e2e > gpurun_out/ev2_config$c.json 2>/dev/null
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 765 --csv \
  --log-file gpurun_out/ev2_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in attn_mma_stream score_signhash compact_quota gather_engine_tma; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 200 -c 1 \
    -o /tmp/ev2_$k -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  ncu -i /tmp/ev2_$k.ncu-rep --page details --csv > gpurun_out/ev2_ncu_${k}_details.csv 2>&1
done
ls -la gpurun_out/ev2_*
