# four GPUs: config 5b / 5c at G = 2 and 4 (n = S = G), ncu of config 5d's kernels at G = 1, boundary tests, config 4
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_boundary.py -m gpu -q -p no:cacheprovider > gpurun_out/c5_boundary.log 2>&1; echo boundary rc=$?; tail -2 gpurun_out/c5_boundary.log
for C in 5b 5c; do for G in 2 4; do
timeout 900 python bench.py --gpus $G --config $C --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/fin_c${C}_g$G.json 2> gpurun_out/fin_c${C}_g$G.err; echo c$C g$G rc=$?
done; done
for rep in 1 2; do timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/fin_c4_rep$rep.json 2>/dev/null; echo c4 rc=$?; done
timeout 1200 ncu --set full --clock-control none -k regex:"asp_replay|bsp_update" -s 4 -c 2 -o gpurun_out/fin_ncu_c5d -f python bench.py --config 5d --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu_c5d.log 2>&1; echo ncu5d rc=$?
