set -u
free -g > gpurun_out/r2_c26_free.txt
timeout 900 python bench.py > gpurun_out/r2_c26_default.json 2> gpurun_out/r2_c26_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_c26_reference.json 2> gpurun_out/r2_c26_reference.err
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e"
$B --sigma 0.07 --steps 30 > gpurun_out/r2_c26_sigma0.07.json 2>&1
$B --config 3 --steps 8 > gpurun_out/r2_c26_config3.json 2>&1
$B --config 4 --steps 8 > gpurun_out/r2_c26_config4.json 2>&1
$B --config 4 --batch 4 --layers 4 --steps 8 > gpurun_out/r2_c26_config4_b4l4_alias.json 2>&1
$B --config 4 --batch 4 --layers 4 --steps 8 --no-alias > gpurun_out/r2_c26_config4_b4l4_noalias.json 2>&1
