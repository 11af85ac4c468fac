#!/bin/bash
# One 4-GPU box: the world-4 fuzz programs, then the default bench at G = 4 and G = 2 (GPUs 0,1).
bash tools/fuzz_debug.sh 4 5400 5401 5402 5403 5404 5405 5406 5407 > gpurun_out/fzd4.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 4 > gpurun_out/bench_g4.json 2> gpurun_out/bench_g4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
echo done
