#!/bin/bash
# Bench contract checks: reference arm (N=1 and torchrun N=2), our arm under torchrun N=2 on one
# device (request sharding, functional), default N=1 line.
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/cc_ref1.json 2> gpurun_out/cc_ref1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --impl reference --gpus 2 --steps 4 --warmup 3 > gpurun_out/cc_ref2.json 2> gpurun_out/cc_ref2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --gpus 2 --same-device --batch 4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/cc_ours2.json 2> gpurun_out/cc_ours2.err
