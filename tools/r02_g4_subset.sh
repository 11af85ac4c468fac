# four GPUs, final tree: 4-GPU parity cases (every exchange mode), full-size sampled (modes 1-3, NVLS forced), 8 fuzz
# programs
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "multi_gpu and (full_size or parity or fuzz) and (4] or -4])" > gpurun_out/g4s_suite.log 2>&1; echo suite rc=$?; tail -1 gpurun_out/g4s_suite.log
exit 0
