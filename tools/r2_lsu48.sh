# LSU default 48: GPU tests (long-context + transfer modes), configs[2] and configs[3] default lines
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_lsu48.log 2>&1; tail -1 gpurun_out/gputests_lsu48.log
timeout 900 python bench.py --config 3 --no-e2e > gpurun_out/l48_c2.json 2>/dev/null
timeout 900 python bench.py --config 4 --steps 16 --no-e2e > gpurun_out/l48_c3.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/l48_c1.json 2>/dev/null
