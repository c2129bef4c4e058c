set -u
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c31_gputest.log 2>&1
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e"
$B --steps 40 > gpurun_out/r2_c31_c1_a.json 2>&1
$B --steps 40 > gpurun_out/r2_c31_c1_b.json 2>&1
for c in 16 24 32; do CLO_GATHER_CTAS=$c $B --config 4 --steps 8 > gpurun_out/r2_c31_c4_lsu$c.json 2>&1; done
for c in 16 24 32; do CLO_GATHER_CTAS=$c $B --config 3 --steps 8 > gpurun_out/r2_c31_c3_lsu$c.json 2>&1; done
