# one GPU: single-GPU suite, A/B of the round-1 kernels vs current (same box, interleaved), ncu of config 2 and 3
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/r02e_suite.log 2>&1; echo suite rc=$?; tail -2 gpurun_out/r02e_suite.log
for rep in 1 2; do
for V in cur r01; do
if [ $V = r01 ]; then export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/r01_kernels.so; else unset SS_LIB_VARIANT; fi
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02e_c2_${V}_$rep.json 2>/dev/null; echo c2 $V $rep rc=$?
timeout 300 python bench.py --config 3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/r02e_c3_${V}_$rep.json 2>/dev/null; echo c3 $V $rep rc=$?
done
done
unset SS_LIB_VARIANT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"asp_replay|bsp_update" -s 40 -c 2 -o gpurun_out/r02e_ncu_c2 -f python bench.py --config 2 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r02e_ncu_c2.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"asp_replay|bsp_update" -s 10 -c 2 -o gpurun_out/r02e_ncu_c3 -f python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_ncu_c3.log 2>&1; echo ncu3 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e_launches_c3.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_launches.log 2>&1; echo launches rc=$?
