# one-GPU A/B: replay small-launch form vs streaming only, configs 2 and 3; ncu of config 2
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02d_suite.log 2>&1; echo suite rc=$?; tail -2 gpurun_out/r02d_suite.log
for v in 0 1; do
SS_REPLAY_STREAMING=$v timeout 600 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02d_c2_s$v.json 2>/dev/null; echo c2 s$v rc=$?
SS_REPLAY_STREAMING=$v timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02d_c3_s$v.json 2>/dev/null; echo c3 s$v rc=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:asp_replay -s 20 -c 1 -o gpurun_out/r02d_ncu_c2 -f python bench.py --config 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r02d_ncu_c2.log 2>&1; echo ncu rc=$?
