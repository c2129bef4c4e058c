set -u
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
for c in 128 32; do CLO_LIB=paper_2511_14510_b200/libclo_probe.so CLO_GATHER_CTAS=$c $B > gpurun_out/r2_c7_probe_c$c.txt 2>&1; done
