# gather in-flight shape A/B at configs[1] (same box)
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1; }
echo "default $(run X=1)" > gpurun_out/gshape.txt
echo "1x2 $(run CLO_GATHER_TMA_SHAPE=1,2)" >> gpurun_out/gshape.txt
echo "1x2_96 $(run CLO_GATHER_TMA_SHAPE=1,2 CLO_GATHER_CTAS=96)" >> gpurun_out/gshape.txt
echo "1x2_64 $(run CLO_GATHER_TMA_SHAPE=1,2 CLO_GATHER_CTAS=64)" >> gpurun_out/gshape.txt
echo "148 $(run CLO_GATHER_CTAS=148)" >> gpurun_out/gshape.txt
echo "default2 $(run X=1)" >> gpurun_out/gshape.txt
