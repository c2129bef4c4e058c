set -x
for c in 1 3 4; do timeout 1500 python bench.py --config $c --steps 16 --warmup 3 --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -c 1500 gpurun_out/bench_c$c.json; tail -3 gpurun_out/bench_c$c.err; done
