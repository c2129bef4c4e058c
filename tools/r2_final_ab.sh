# final-tree A/B of the switches around the default (configs[1], same box, alternating)
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1; }
: > gpurun_out/fab.txt
for i in 1 2; do
  echo "default $(run X=1)" >> gpurun_out/fab.txt
  echo "sel2 $(run CLO_SEL_STREAMS=2)" >> gpurun_out/fab.txt
  echo "ctas112 $(run CLO_GATHER_CTAS=112)" >> gpurun_out/fab.txt
  echo "ctas136 $(run CLO_GATHER_CTAS=136)" >> gpurun_out/fab.txt
done
