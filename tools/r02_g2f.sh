# two GPUs: single-GPU suite, 2-GPU parity (fused modes incl. pull, capture, fuzz), benches G = 1 (configs 2, 3) and
# G = 2 (configs 3, 5a)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/r02f_suite1.log 2>&1; echo suite1 rc=$?; tail -2 gpurun_out/r02f_suite1.log
timeout 1800 python -m pytest tests/test_multi_gpu.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "multi_gpu and not full_size and (2] or -2])" > gpurun_out/r02f_suite2.log 2>&1; echo suite2 rc=$?; tail -3 gpurun_out/r02f_suite2.log
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02f_c2_g1.json 2>/dev/null; echo c2 rc=$?
timeout 300 python bench.py --config 3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02f_c3_g1.json 2>/dev/null; echo c3 rc=$?
timeout 600 python bench.py --gpus 2 --config 3 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02f_c3_g2.json 2>/dev/null; echo c3g2 rc=$?
timeout 600 python bench.py --gpus 2 --config 5a --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02f_c5a_g2.json 2>/dev/null; echo c5ag2 rc=$?
timeout 600 python bench.py --gpus 2 --config 2 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02f_c2_g2.json 2>/dev/null; echo c2g2 rc=$?
