set -u
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 40"
for r in 1 2 3; do
  $B > gpurun_out/r2_c33_def_$r.json 2>&1
  CLO_ATTN_NOTMA=1 $B > gpurun_out/r2_c33_notma_$r.json 2>&1
  CLO_SCORE=lsu $B > gpurun_out/r2_c33_lsuscore_$r.json 2>&1
done
