set -x
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --steps 64 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['step_ms'], d['hit_ratio'], d['e2e']['value'], d['per_kernel_ms'])"; done
