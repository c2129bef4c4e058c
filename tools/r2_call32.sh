set -u
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 40"
for r in 1 2 3; do
  $B > gpurun_out/r2_c32_new_$r.json 2>&1
  CLO_LIB=paper_2511_14510_b200/libclo_prev.so $B > gpurun_out/r2_c32_prev_$r.json 2>&1
done
B4="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8"
for r in 1 2; do
  CLO_GATHER_CTAS=24 $B4 --config 4 > gpurun_out/r2_c32_c4_lsu24_$r.json 2>&1
  $B4 --config 4 > gpurun_out/r2_c32_c4_lsu48_$r.json 2>&1
done
