# one-GPU: parity suite (single GPU), config 2 / 3 bench, ncu of config 2's window kernel
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/r02_g1c_suite.log 2>&1; echo suite rc=$?; tail -3 gpurun_out/r02_g1c_suite.log
timeout 600 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02c_bench_c2.json 2> gpurun_out/r02c_bench_c2.err; echo bench2 rc=$?
timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02c_bench_c3.json 2> gpurun_out/r02c_bench_c3.err; echo bench3 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:asp_replay -s 20 -c 1 -o gpurun_out/r02c_ncu_c2 -f python bench.py --config 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r02c_ncu_c2.log 2>&1; echo ncu rc=$?
