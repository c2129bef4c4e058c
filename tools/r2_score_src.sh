# score kernel: ncu --set full with source export (a layer-0 persistent launch: 128 items), and selection-stream priority A/B
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_signhash -s 20 -c 1 \
  -o /tmp/sc -f python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/sc.ncu-rep --page details --csv > gpurun_out/sc_details.csv 2>&1
ncu -i /tmp/sc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/sc_source.csv 2>&1
for p in high mid; do
  CLO_SEL_PRIO=$p timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/prio_$p.json 2>/dev/null
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/prio_default.json 2>/dev/null
