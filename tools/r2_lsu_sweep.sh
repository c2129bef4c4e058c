# LSU gather grid (long contexts: per-head host regions > 48 MiB) at configs[2] and configs[3]
run() { env "$@" timeout 900 python bench.py --no-cpu-baseline --no-e2e "${ARGS[@]}" 2>/dev/null | tail -1; }
: > gpurun_out/lsweep.txt
ARGS=(--config 3)
for i in 1 2; do for c in 16 24 40; do echo "c2_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/lsweep.txt; done; done
ARGS=(--config 4 --steps 16)
for c in 24 40; do echo "c3_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/lsweep.txt; done
