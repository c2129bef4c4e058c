B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
CLO_LIB=paper_2511_14510_b200/libclo_probe.so CLO_GATHER_CTAS=8 $B > gpurun_out/r2_c21_probe_c8.txt 2>&1
CLO_LIB=paper_2511_14510_b200/libclo_probe.so $B > gpurun_out/r2_c21_probe_c128.txt 2>&1
