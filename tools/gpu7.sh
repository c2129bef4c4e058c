set -x
timeout 600 python bench_gather.py --reps 5 2>&1 | tail -12
timeout 600 python bench_gather.py --reps 3 --ctas 148 --rows 2048,16384 2>&1 | tail -3
timeout 600 python bench_gather.py --reps 3 --ctas 296 --rows 2048,16384 2>&1 | tail -3
