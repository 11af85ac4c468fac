# two GPUs after the event-table change: 2-GPU parity subset (full-size sampled included), default single-GPU line,
# 2-GPU config 3 line
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_multi_gpu.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "multi_gpu and (2] or -2])" > gpurun_out/fc_suite2.log 2>&1; echo suite2 rc=$?; tail -1 gpurun_out/fc_suite2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --steps 2000 --warmup 20 > gpurun_out/fc_c3_g1.json 2> gpurun_out/fc_c3_g1.err; echo c3 rc=$?
timeout 900 python bench.py --gpus 2 --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/fc_c3_g2.json 2> gpurun_out/fc_c3_g2.err; echo c3g2 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fc_launches_c3.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fc_launches.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"asp_replay|bsp_update" -s 10 -c 2 -o gpurun_out/fc_ncu_c3 -f python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fc_ncu_c3.log 2>&1; echo ncu3 rc=$?
exit 0
