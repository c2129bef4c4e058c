set -x
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_shard.py -q -x 2>&1 | tail -3
run() { timeout 900 python bench.py --config 2 "$@" --steps 32 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['rooflines']['gather_zero_copy']; print('$*', round(d['value'],1), d['step_ms'], 'gather GB/s', round(r['achieved'],1), 'pcie in step', round(d['pcie_gather_gbs_in_step'],1), d['kernels_per_step'])"; }
run
run --batch 4 --ctx 524288
