# default TMA gather grid 112: GPU tests, configs[1] x2, configs[0], smoke
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_112.log 2>&1; tail -1 gpurun_out/gputests_112.log
timeout 600 python bench.py > gpurun_out/c112_a.json 2> gpurun_out/c112_a.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/c112_b.json 2> /dev/null
timeout 600 python bench.py --config 1 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/c112_c0.json 2> /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_112.log 2>&1; tail -1 gpurun_out/smoke_112.log
