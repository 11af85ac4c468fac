# two GPUs: an extended fuzz run — 512 seeded single-GPU programs and 24 per world size at 2 GPUs
cd $GRAFT_REPO_ROOT
SS_FUZZ_CASES=512 timeout 1200 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "bit_exact" > gpurun_out/fz_single.log 2>&1; echo single rc=$?; tail -1 gpurun_out/fz_single.log
SS_FUZZ_MULTI_CASES=24 timeout 1200 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "multi_gpu and -2]" > gpurun_out/fz_multi2.log 2>&1; echo multi rc=$?; tail -1 gpurun_out/fz_multi2.log
exit 0
