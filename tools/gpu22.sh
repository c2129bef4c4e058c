#!/bin/bash
# Fused head-output exchange: GPU tests + a 2-rank functional bench on one device.
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_shard.py -x -q > gpurun_out/p22_tests.log 2>&1
echo "rc=$?" >> gpurun_out/p22_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --config 4 --same-device --ctx 65536 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/p22_bench_2rank.log 2>&1
echo "rc=$?" >> gpurun_out/p22_bench_2rank.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --config 4 --same-device --ctx 65536 --steps 8 --warmup 3 --no-cpu-baseline --allgather nccl > gpurun_out/p22_bench_2rank_nccl.log 2>&1
echo "rc=$?" >> gpurun_out/p22_bench_2rank_nccl.log
