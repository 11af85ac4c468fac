#!/bin/bash
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r_c3.json 2> gpurun_out/r_c3.err; echo "c3 $?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config 2 --steps 3000 --warmup 50 --no-e2e --no-cpu-baseline > gpurun_out/r_c2.json 2> gpurun_out/r_c2.err; echo "c2 $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 \
  bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r_g2.json 2> gpurun_out/r_g2.err; echo "g2 $?"
