# attention cluster merge: GPU tests, then configs[2]/configs[1] A/B (CLO_ATTN_CLUSTER=0 = global merge)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests2.log 2>&1; tail -3 gpurun_out/gputests2.log
for c in 3 2; do
 for a in 1 0; do
  CLO_ATTN_CLUSTER=$a timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/cl_c${c}_a${a}.json 2> gpurun_out/cl_c${c}_a${a}.err
 done
done
CLO_BENCH_SPANS=gpurun_out/spans_c2_cluster.json timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/cl_c3_spans.json 2>/dev/null
