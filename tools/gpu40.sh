#!/bin/bash
# ncu of the decode-step selection chain kernels (prepare, score, threshold, compact, reconcile, append).
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prepare_kernel|score_signhash|threshold_signhash|compact_kernel|reconcile_kernel|append_kernel" \
  -s 400 -c 12 -o gpurun_out/p40_sel -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p40_ncu.log 2>&1
