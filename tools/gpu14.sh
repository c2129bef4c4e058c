set -x
for c in 48 148 592; do timeout 600 python bench_gather.py --reps 3 --n 1048576 --rows 2048 --heads 8 --ctas $c 2>&1 | grep rows_per | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep n=1M ctas $c', round(d['lsu_gbs'],1), round(d['tma_gbs'],1))"; done
run() { timeout 900 python bench.py --config 2 --batch 4 --ctx 524288 --steps 16 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['rooflines']['gather_zero_copy']; print('$1', round(d['value'],1), 'gather GB/s', round(r['achieved'],1), 'pcie in step', round(d['pcie_gather_gbs_in_step'],1))"; }
for c in 48 148 296 592; do CLO_GATHER_CTAS=$c run ctas=$c; done
