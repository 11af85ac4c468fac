# one-GPU: full single-GPU suite (no -x), ncu full capture of config 2's window kernel
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/r02_g1_suite2.log 2>&1; echo suite rc=$?; tail -5 gpurun_out/r02_g1_suite2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:asp_replay -s 20 -c 2 -o gpurun_out/r02_ncu_c2 -f python bench.py --config 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_c2.log 2>&1; echo ncu rc=$?
