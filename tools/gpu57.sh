#!/bin/bash
# Footprint vs heads touched: 8 heads over 4M rows (17 GB) vs 32 heads over 1M (17 GB), and 2 heads over 16M (17 GB).
timeout 900 python bench_gather.py --n 4194304 --heads 8 --rows 2048,8192 --reps 3 --skip-cpu > gpurun_out/p57_h8_n4m.jsonl 2>&1
timeout 900 python bench_gather.py --n 16777216 --heads 2 --rows 8192,32768 --reps 3 --skip-cpu > gpurun_out/p57_h2_n16m.jsonl 2>&1
timeout 900 python bench_gather.py --n 2097152 --heads 8 --rows 2048,8192 --reps 3 --skip-cpu > gpurun_out/p57_h8_n2m.jsonl 2>&1
