set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c11_gputest.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20"
NT=paper_2511_14510_b200/libclo_nt.so
for c in 48 128; do
  CLO_GATHER_CTAS=$c $B > gpurun_out/r2_c11_trig_ov_$c.json 2>&1
  CLO_GATHER_CTAS=$c CLO_GATHER_OVERLAP=0 $B > gpurun_out/r2_c11_trig_noov_$c.json 2>&1
  CLO_LIB=$NT CLO_GATHER_CTAS=$c $B > gpurun_out/r2_c11_nt_ov_$c.json 2>&1
  CLO_LIB=$NT CLO_GATHER_CTAS=$c CLO_GATHER_OVERLAP=0 $B > gpurun_out/r2_c11_nt_noov_$c.json 2>&1
  CLO_PDL=0 CLO_GATHER_CTAS=$c $B > gpurun_out/r2_c11_nopdl_$c.json 2>&1
done
