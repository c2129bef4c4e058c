#!/bin/bash
for h in 16 32 64; do
timeout 900 python bench_gather.py --n 1048576 --heads $h --rows 2048 --reps 3 --skip-cpu > gpurun_out/p56_g1m_h$h.jsonl 2>&1
done
timeout 900 python bench_gather.py --n 1048576 --heads 64 --rows 2048 --reps 3 --skip-cpu --huge > gpurun_out/p56_g1m_h64_huge.jsonl 2>&1
