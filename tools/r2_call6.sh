set -u
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
run() { tag=$1; shift; env "$@" CLO_BENCH_SPANS=gpurun_out/r2_c6_spans_$tag.json $B > gpurun_out/r2_c6_$tag.json 2>&1; }
run t16s4 CLO_GATHER_CTAS=16 CLO_GATHER_TMA_SHAPE=1,4
run t24s3 CLO_GATHER_CTAS=24 CLO_GATHER_TMA_SHAPE=1,3
run t32s2 CLO_GATHER_CTAS=32 CLO_GATHER_TMA_SHAPE=1,2
run t32s3 CLO_GATHER_CTAS=32 CLO_GATHER_TMA_SHAPE=1,3
run t8w2s4 CLO_GATHER_CTAS=8 CLO_GATHER_TMA_SHAPE=2,4
run lsu48 CLO_GATHER=lsu CLO_GATHER_CTAS=48
run lsu96 CLO_GATHER=lsu CLO_GATHER_CTAS=96
