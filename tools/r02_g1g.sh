# one GPU: single-GPU suite with the register form, config-2 A/B of the window kernel's small forms
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/r02g_suite.log 2>&1; echo suite rc=$?; tail -2 gpurun_out/r02g_suite.log
for rep in 1 2; do for V in 1 0; do
SS_REPLAY_SMALL=$V timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r02g_c2_s${V}_$rep.json 2>/dev/null; echo c2 s$V rc=$?
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"asp_replay" -s 40 -c 1 -o gpurun_out/r02g_ncu_c2 -f python bench.py --config 2 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r02g_ncu_c2.log 2>&1; echo ncu2 rc=$?
