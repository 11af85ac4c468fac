# two GPUs: pull-mode (fused 3) parity cases + config 5a bench in mode 3 vs mode 1
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q -p no:cacheprovider -x -k "pull or (edge and 3]) or (capture and 3]) or (host_buffers and 3])" > gpurun_out/r02_g2pull_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r02_g2pull_tests.log
for F in 3 1; do
timeout 600 python bench.py --gpus 2 --config 5a --fused $F --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02_c5a_g2_f$F.json 2> gpurun_out/r02_c5a_g2_f$F.err; echo c5a f$F rc=$?
done
