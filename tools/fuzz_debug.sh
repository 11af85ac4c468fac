#!/bin/bash
# Runs multi-GPU fuzz programs (tests/dist_fuzz_worker.py) one by one with a short timeout, keeping their outputs:
#   bash tools/fuzz_debug.sh G seed...   -> gpurun_out/fz_<seed>/rank*.npz, gpurun_out/fz_<seed>.log
G=$1; shift
for s in "$@"; do
  mkdir -p gpurun_out/fz_$s
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port $((29500 + s % 1000)) tests/dist_fuzz_worker.py --out gpurun_out/fz_$s \
    --seed $s > gpurun_out/fz_$s.log 2>&1
  echo "seed $s rc=$?"
done
