#!/bin/bash
# Full GPU suite + default bench (with timeline breakdown) after the graph-mode refactor.
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p37_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p37_tests.log
timeout 600 python bench.py > gpurun_out/p37_bench.json 2> gpurun_out/p37_bench.err
