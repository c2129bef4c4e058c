#!/bin/bash
t() { timeout 600 python -m pytest tests/test_gpu_exchange.py -x -q -k "in_process" > gpurun_out/p50_$1.log 2>&1; echo "rc=$?" >> gpurun_out/p50_$1.log; }
CLO_LIB=$PWD/paper_2511_14510_b200/libclo_head.so t head
t cur
CLO_EXCHANGE_TIMEOUT_MS=90000 t cur_long
