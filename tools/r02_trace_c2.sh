# two GPUs: SS_TRACE breakdown of config 2's fused kernels (bench launch configuration), default and mode 3
cd $GRAFT_REPO_ROOT
SS_TRACE=gpurun_out/r02_trace_c2_g2 timeout 300 python bench.py --gpus 2 --config 2 --steps 600 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02_trace_c2_g2.json 2>/dev/null; echo rc=$?
python tools/trace_report.py gpurun_out/r02_trace_c2_g2 --skip 100 > gpurun_out/r02_trace_c2_g2.txt 2>&1; cat gpurun_out/r02_trace_c2_g2.txt
SS_TRACE=gpurun_out/r02_trace_c2_g2_f3 timeout 300 python bench.py --gpus 2 --config 2 --fused 3 --steps 600 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02_trace_c2_g2_f3.json 2>/dev/null; echo rc=$?
python tools/trace_report.py gpurun_out/r02_trace_c2_g2_f3 --skip 100 > gpurun_out/r02_trace_c2_g2_f3.txt 2>&1; cat gpurun_out/r02_trace_c2_g2_f3.txt
