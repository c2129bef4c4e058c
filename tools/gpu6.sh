set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
CLO_ATTN_LANES=16 timeout 900 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -3
for L in 8 16; do CLO_ATTN_LANES=$L timeout 900 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes',$L, d['value'], d['per_kernel_ms'])"; done
