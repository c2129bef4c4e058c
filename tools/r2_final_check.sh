# final tree: GPU tests + smoke
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; tail -1 gpurun_out/gputests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
