set -u
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prepare_kernel|append_kernel|reconcile_kernel" -s 400 -c 6 -o gpurun_out/r2_lat -f $B > gpurun_out/r2_lat.log 2>&1
echo rc=$?
