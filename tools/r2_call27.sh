set -u
timeout 900 python -m pytest tests/test_gpu_output_error.py -x -q > gpurun_out/r2_c27_oerr.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c27_gputest.log 2>&1
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e"
$B --layers 8 --steps 20 > gpurun_out/r2_c27_l8_alias.json 2>&1
$B --layers 8 --steps 20 --no-alias > gpurun_out/r2_c27_l8_noalias.json 2>&1
$B --config 4 --layers 3 --steps 8 > gpurun_out/r2_c27_c4l3_alias.json 2>&1
$B --config 4 --layers 3 --steps 8 --no-alias > gpurun_out/r2_c27_c4l3_noalias.json 2>&1
