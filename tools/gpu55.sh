#!/bin/bash
# Large host stores: GPU TLB reach with 4 KiB vs 2 MiB host pages.
timeout 600 python bench_gather.py --n 1048576 --heads 8 --rows 2048,8192 --skip-cpu > gpurun_out/p55_g1m.jsonl 2>&1
timeout 600 python bench_gather.py --n 1048576 --heads 8 --rows 2048,8192 --skip-cpu --huge > gpurun_out/p55_g1m_huge.jsonl 2>&1
timeout 1500 python bench.py --config 4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --huge > gpurun_out/p55_c4_huge.json 2> gpurun_out/p55_c4_huge.err
timeout 900 python bench.py --steps 16 --no-e2e --no-cpu-baseline --huge > gpurun_out/p55_c2_huge.json 2> gpurun_out/p55_c2_huge.err
