set -u
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8"
for cfg in 4 3; do
  $B --config $cfg > gpurun_out/r2_c36_c${cfg}_def.json 2>&1
  CLO_GATHER=wide CLO_GATHER_CTAS=20 CLO_GATHER_WIDE=3 $B --config $cfg > gpurun_out/r2_c36_c${cfg}_w20_1024.json 2>&1
  CLO_GATHER=wide CLO_GATHER_CTAS=20 $B --config $cfg > gpurun_out/r2_c36_c${cfg}_w20_512.json 2>&1
  CLO_GATHER=wide CLO_GATHER_CTAS=16 CLO_GATHER_WIDE=3 $B --config $cfg > gpurun_out/r2_c36_c${cfg}_w16_1024.json 2>&1
  CLO_GATHER=tma $B --config $cfg > gpurun_out/r2_c36_c${cfg}_tma128.json 2>&1
done
