set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --ctx 16384 --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | tail -20
timeout 900 python bench.py --steps 16 --warmup 3 --no-cpu-baseline 2>&1 | tail -20
