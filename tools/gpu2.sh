set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 900 python bench.py --steps 32 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_engine_kernel -s 40 -c 2 -o gpurun_out/prof_attn -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_signhash -s 20 -c 2 -o gpurun_out/prof_score -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_score.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_engine -s 20 -c 2 -o gpurun_out/prof_gather -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gather.log 2>&1
ls -la gpurun_out
