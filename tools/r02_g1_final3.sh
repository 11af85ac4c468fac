# one GPU: single-GPU suite and the config-2 line after the lone-superstep kernel choice
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/f3_suite.log 2>&1; echo suite rc=$?; tail -1 gpurun_out/f3_suite.log
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline > gpurun_out/f3_c2_g1.json 2> gpurun_out/f3_c2_g1.err; echo c2 rc=$?
timeout 300 python bench.py --config 5a --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/f3_c5a_g1.json 2> /dev/null; echo c5a rc=$?
exit 0
