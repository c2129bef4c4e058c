set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c10_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
for c in 128 64 48 32; do CLO_GATHER_CTAS=$c $B > gpurun_out/r2_c10_ctas_$c.json 2>&1; done
CLO_PDL=0 CLO_GATHER_CTAS=48 $B > gpurun_out/r2_c10_nopdl_48.json 2>&1
