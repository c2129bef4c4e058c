set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 900 python bench.py --steps 32 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
