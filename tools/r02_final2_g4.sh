# four GPUs, final: full -m gpu suite at the committed tree, then the multi-GPU bench lines (G = 4 and 2)
cd $GRAFT_REPO_ROOT
timeout 3300 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/f2_g4_suite.log 2>&1; echo suite rc=$?; tail -3 gpurun_out/f2_g4_suite.log
for G in 4 2; do
timeout 900 python bench.py --gpus $G --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/f2_c3_g$G.json 2> gpurun_out/f2_c3_g$G.err; echo c3 g$G rc=$?
timeout 600 python bench.py --gpus $G --config 2 --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/f2_c2_g$G.json 2> gpurun_out/f2_c2_g$G.err; echo c2 g$G rc=$?
timeout 900 python bench.py --gpus $G --config 5a --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/f2_c5a_g$G.json 2> gpurun_out/f2_c5a_g$G.err; echo c5a g$G rc=$?
done
