set -x
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag
for n in 131072 524288 1048576; do timeout 600 python bench_gather.py --reps 3 --n $n --rows 2048 --heads 16 2>&1 | grep rows_per | cut -c1-400; timeout 600 python bench_gather.py --reps 3 --n $n --rows 2048 --heads 16 --huge 2>&1 | grep rows_per | cut -c1-400; done
grep -i huge /proc/meminfo
