#!/bin/bash
n() { timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"score_signhash" -s 300 -c 20 --csv --log-file gpurun_out/p53_$1.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; }
n base
CLO_SCORE_AGG=1 n agg
CLO_SCORE_GRID=1184 n g1184
CLO_SCORE_AGG=1 CLO_SCORE_GRID=1184 n agg_g1184
CLO_SCORE=lsu n lsu
