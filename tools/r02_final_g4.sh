# four GPUs, round-2 final: the full -m gpu suite (1-, 2- and 4-GPU tests), bench lines at G = 2 and 4 for configs
# 3, 2, 5a, 5d (default exchange), config 3 in every exchange mode at G = 4, NCCL mode with NCCL's algorithm logged
cd $GRAFT_REPO_ROOT
timeout 3300 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/fin_g4_suite.log 2>&1; echo suite rc=$?; tail -3 gpurun_out/fin_g4_suite.log
for G in 4 2; do
timeout 900 python bench.py --gpus $G --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/fin_c3_g$G.json 2> gpurun_out/fin_c3_g$G.err; echo c3 g$G rc=$?
timeout 600 python bench.py --gpus $G --config 2 --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/fin_c2_g$G.json 2> gpurun_out/fin_c2_g$G.err; echo c2 g$G rc=$?
timeout 900 python bench.py --gpus $G --config 5a --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/fin_c5a_g$G.json 2> gpurun_out/fin_c5a_g$G.err; echo c5a g$G rc=$?
timeout 900 python bench.py --gpus $G --config 5d --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin_c5d_g$G.json 2> gpurun_out/fin_c5d_g$G.err; echo c5d g$G rc=$?
done
for F in 0 1 3; do
timeout 900 python bench.py --gpus 4 --fused $F --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/fin_c3_g4_f$F.json 2> gpurun_out/fin_c3_g4_f$F.err; echo c3 g4 f$F rc=$?
done
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 900 python bench.py --gpus 4 --config 5a --fused 0 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/fin_c5a_g4_nccl.json 2> gpurun_out/fin_c5a_g4_nccl.err; echo nccl rc=$?
timeout 900 python bench.py --gpus 4 --config 3 --workload > gpurun_out/fin_wl3_g4.json 2> gpurun_out/fin_wl3_g4.err; echo wl3 g4 rc=$?
