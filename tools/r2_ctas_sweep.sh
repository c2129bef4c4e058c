# TMA gather grid sweep around the default at the final tree (configs[1] x2 each, configs[0] and configs[2] at the best candidates)
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e "${ARGS[@]}" 2>/dev/null | tail -1; }
: > gpurun_out/csweep.txt
ARGS=()
for i in 1 2; do
  for c in 96 104 112 120 128; do echo "c2_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/csweep.txt; done
done
ARGS=(--config 1 --steps 200 --warmup 5)
for c in 112 128; do echo "c0_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/csweep.txt; done
ARGS=(--config 3)
for c in 112 128; do echo "c3_$c $(run CLO_GATHER_CTAS=$c)" >> gpurun_out/csweep.txt; done
