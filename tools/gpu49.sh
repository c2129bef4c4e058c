#!/bin/bash
t() { timeout 600 python -m pytest tests/test_gpu_exchange.py -x -q -k "in_process and 4" > gpurun_out/p49_$1.log 2>&1; echo "rc=$?" >> gpurun_out/p49_$1.log; }
t default
CLO_ATTN_REGCAP=184 t cap
CLO_ATTN=tma t tma
CLO_ATTN_SHAPE=4x3x1x32 t small
