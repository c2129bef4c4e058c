#!/bin/bash
# Every BASELINE config once (1 GPU): configs[0] 32K always-miss B=1, configs[2] Qwen 512K B=4
# plan_partition, configs[3] 1M B=8 (unsharded on one GPU).
timeout 900 python bench.py --config 1 --steps 8 --warmup 3 --no-e2e > gpurun_out/p54_c1.json 2> gpurun_out/p54_c1.err
timeout 1200 python bench.py --config 3 --steps 8 --warmup 3 --no-e2e > gpurun_out/p54_c3.json 2> gpurun_out/p54_c3.err
timeout 1500 python bench.py --config 4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p54_c4.json 2> gpurun_out/p54_c4.err
