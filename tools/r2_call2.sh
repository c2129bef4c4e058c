set -u
B="timeout 600 python bench.py --no-cpu-baseline"
CLO_BENCH_SPANS=gpurun_out/r2_spans.json $B --steps 20 --no-e2e > gpurun_out/r2_spans_bench.json 2>&1
for v in 16384 32768; do $B --steps 30 --no-e2e --victim-rows $v > gpurun_out/r2_victim_$v.json 2>&1; done
for s in 0.02 0.1 0.2 0.35; do $B --steps 30 --no-e2e --sigma $s > gpurun_out/r2_sigma_$s.json 2>&1; done
$B --config 1 --steps 20 > gpurun_out/r2_config1.json 2>&1
$B --kv-dtype f32 --steps 30 --no-e2e > gpurun_out/r2_f32.json 2>&1
