set -u
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c29_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 40"
for r in 1 2; do
for m in thr 0 all; do CLO_CHAIN_SELECT=$m $B > gpurun_out/r2_c29_${m}_$r.json 2>&1; done
done
