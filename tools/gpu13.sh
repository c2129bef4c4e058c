set -x
run() { timeout 900 python bench.py --config 2 "$@" --steps 16 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['rooflines']['gather_zero_copy']; print('$*', round(d['value'],1), 'hit', round(d['hit_ratio'],3), 'gather GB/s', round(r['achieved'],1), 'gather ms', d['per_kernel_ms']['gather_zero_copy'], 'pcie in step', round(d['pcie_gather_gbs_in_step'],1))"; }
run --batch 4
run --batch 16 --ctx 524288
run --batch 4 --ctx 524288
run --batch 64 --ctx 32768
