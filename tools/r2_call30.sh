set -u
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8"
$B --config 3 > gpurun_out/r2_c30_c3_default.json 2>&1
CLO_ATTN_ALIGN=0 $B --config 3 > gpurun_out/r2_c30_c3_noalign.json 2>&1
CLO_ATTN_SHAPE=4x3x2x16 $B --config 3 > gpurun_out/r2_c30_c3_4x3x2.json 2>&1
CLO_ATTN_SHAPE=4x6x1x16 $B --config 3 > gpurun_out/r2_c30_c3_4x6x1.json 2>&1
CLO_GATHER=tma $B --config 3 > gpurun_out/r2_c30_c3_tma.json 2>&1
CLO_GATHER_CTAS=96 $B --config 3 > gpurun_out/r2_c30_c3_lsu96.json 2>&1
$B --config 4 > gpurun_out/r2_c30_c4_default.json 2>&1
CLO_GATHER=tma $B --config 4 > gpurun_out/r2_c30_c4_tma.json 2>&1
CLO_GATHER_CTAS=96 $B --config 4 > gpurun_out/r2_c30_c4_lsu96.json 2>&1
CLO_GATHER_CTAS=24 $B --config 4 > gpurun_out/r2_c30_c4_lsu24.json 2>&1
