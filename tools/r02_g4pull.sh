# four GPUs: pull-mode parity (all pull cases, edge layouts, capture, host buffers, full size), NVLS forced full size;
# A/B of the BSP exchange forms on configs 5a and 3
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multi_gpu.py -m gpu -q -p no:cacheprovider -k "pull or 3] or 3-0] or 1-1]" > gpurun_out/r02_g4pull_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r02_g4pull_tests.log
SS_PULL_TMA=1 timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q -p no:cacheprovider -k "pull or 3-0]" > gpurun_out/r02_g4pull_tma_tests.log 2>&1; echo tma tests rc=$?; tail -3 gpurun_out/r02_g4pull_tma_tests.log
for C in 5a 3; do
for F in 1 2 3; do
timeout 600 python bench.py --gpus 4 --config $C --fused $F --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02_c${C}_g4_f$F.json 2> gpurun_out/r02_c${C}_g4_f$F.err; echo c$C f$F rc=$?
done
SS_PULL_TMA=1 timeout 600 python bench.py --gpus 4 --config $C --fused 3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02_c${C}_g4_f3tma.json 2> gpurun_out/r02_c${C}_g4_f3tma.err; echo c$C f3tma rc=$?
done
