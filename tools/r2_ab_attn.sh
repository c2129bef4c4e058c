set -x
for c in 2 3; do
 for a in 1 0; do
  CLO_ATTN_ALIGN=$a timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/attn_c${c}_a${a}.json 2> gpurun_out/attn_c${c}_a${a}.err
 done
done
