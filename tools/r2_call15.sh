B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
CLO_LIB=paper_2511_14510_b200/libclo_probe.so $B > gpurun_out/r2_c15_probe.txt 2>&1
