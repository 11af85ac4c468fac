# two GPUs: graph capture without per-kernel end barriers — capture tests (even and odd exchange counts), config 2
# and 3 lines (graph timing) at G = 2
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q -p no:cacheprovider -k "graph_capture and 2]" > gpurun_out/gr_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gr_tests.log
timeout 600 python bench.py --gpus 2 --config 2 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/gr_c2_g2.json 2>/dev/null; echo c2 rc=$?
timeout 600 python bench.py --gpus 2 --config 3 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/gr_c3_g2.json 2>/dev/null; echo c3 rc=$?
exit 0
