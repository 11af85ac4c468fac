# two GPUs: fused kernels without PDL — parity subset and config 2 / 3 lines
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_multi_gpu.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x -k "(parity or fuzz or capture) and (2] or -2])" > gpurun_out/np_suite2.log 2>&1; echo suite2 rc=$?; tail -2 gpurun_out/np_suite2.log
timeout 600 python bench.py --gpus 2 --config 2 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/np_c2_g2.json 2>/dev/null; echo c2 rc=$?
timeout 600 python bench.py --gpus 2 --config 3 --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/np_c3_g2.json 2>/dev/null; echo c3 rc=$?
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/np_c2_g1.json 2>/dev/null; echo c2g1 rc=$?
