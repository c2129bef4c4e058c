# LSU gather 48 vs 64 CTAs at configs[3] and configs[2], alternating on one box
run() { env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e "${ARGS[@]}" 2>/dev/null | tail -1; }
: > gpurun_out/lsweep3.txt
ARGS=(--config 4 --steps 16)
for c in 48 64 48 64; do echo "c3_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/lsweep3.txt; done
ARGS=(--config 3)
for c in 48 64; do echo "c2_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/lsweep3.txt; done
