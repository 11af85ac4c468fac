# four GPUs: 8 more seeded fuzz programs at world 4 (cases 8-15) on the final tree
cd $GRAFT_REPO_ROOT
SS_FUZZ_MULTI_CASES=16 timeout 800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "multi_gpu and (8-4 or 9-4 or 10-4 or 11-4 or 12-4 or 13-4 or 14-4 or 15-4)" > gpurun_out/fz4.log 2>&1; echo rc=$?; tail -1 gpurun_out/fz4.log
exit 0
