# LSU gather grid, second pass (configs[2] 40/48/64, configs[3] 40/48)
run() { env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e "${ARGS[@]}" 2>/dev/null | tail -1; }
: > gpurun_out/lsweep2.txt
ARGS=(--config 3)
for c in 40 48 64 40 48 64; do echo "c2_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/lsweep2.txt; done
ARGS=(--config 4 --steps 16)
for c in 40 48; do echo "c3_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/lsweep2.txt; done
