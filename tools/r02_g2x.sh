# two GPUs: one-kernel ASP exchange — 2-GPU parity subset, config 2 / 3 / 5a benches, config-2 trace
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_multi_gpu.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x -k "multi_gpu and (2] or -2])" > gpurun_out/x_suite2.log 2>&1; echo suite2 rc=$?; tail -3 gpurun_out/x_suite2.log
timeout 600 python bench.py --gpus 2 --config 2 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/x_c2_g2.json 2>/dev/null; echo c2g2 rc=$?
timeout 600 python bench.py --gpus 2 --config 3 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/x_c3_g2.json 2>/dev/null; echo c3g2 rc=$?
timeout 600 python bench.py --gpus 2 --config 5a --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/x_c5a_g2.json 2>/dev/null; echo c5ag2 rc=$?
SS_TRACE=gpurun_out/x_trace_c2_g2 timeout 300 python bench.py --gpus 2 --config 2 --steps 600 --warmup 20 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo trace rc=$?
python tools/trace_report.py gpurun_out/x_trace_c2_g2 --skip 100 > gpurun_out/x_trace_c2_g2.txt 2>&1; cat gpurun_out/x_trace_c2_g2.txt
