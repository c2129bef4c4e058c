set -u
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
for g in 296 444 592 1184; do CLO_SCORE_GRID=$g $B > gpurun_out/r2_c25_grid$g.json 2>&1; done
