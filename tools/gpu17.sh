set -x
CLO_TRANSFER=events timeout 600 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2
for h in 4 16; do timeout 600 python bench_gather.py --reps 3 --n 524288 --rows 1900 --heads $h --ctas 48 2>&1 | grep rows_per | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep n=512K heads $h ctas 48', round(d['lsu_gbs'],1))"; done
timeout 900 ncu --set full --clock-control none -k regex:"gather_engine" -s 40 -c 3 -o gpurun_out/prof_g512 -f python bench.py --config 2 --batch 4 --ctx 524288 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_g512.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gather_engine" -s 40 -c 3 -o gpurun_out/prof_g128 -f python bench.py --config 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_g128.log 2>&1
