# four GPUs: NVLS ld_reduce microbench, the full -m gpu suite (1-, 2- and 4-GPU tests), benches at G = 1, 2, 4
cd $GRAFT_REPO_ROOT
export LD_LIBRARY_PATH=
timeout 300 ./tools/nvls_reduce_bench 32 > gpurun_out/r02_nvls_reduce_32.txt 2>&1; echo nvls32 rc=$?
timeout 300 ./tools/nvls_reduce_bench 128 > gpurun_out/r02_nvls_reduce_128.txt 2>&1; echo nvls128 rc=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 ./tools/nvls_reduce_bench 32 > gpurun_out/r02_nvls_reduce_32_g2.txt 2>&1; echo nvls32g2 rc=$?
unset LD_LIBRARY_PATH
git rev-parse HEAD > gpurun_out/r02_g4_head.txt 2>/dev/null
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r02_g4_suite.log 2>&1; echo suite rc=$?; tail -3 gpurun_out/r02_g4_suite.log
for G in 4 2 1; do
timeout 600 python bench.py --gpus $G --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/r02_bench_c3_g$G.json 2> gpurun_out/r02_bench_c3_g$G.err; echo c3 g$G rc=$?
timeout 600 python bench.py --gpus $G --config 2 --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c2_g$G.json 2> gpurun_out/r02_bench_c2_g$G.err; echo c2 g$G rc=$?
done
