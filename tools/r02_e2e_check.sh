# two GPUs: e2e after the staging warm-up — config 3 at G = 2 twice, the default single-GPU line once
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
timeout 600 python bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/e2c_g2_$rep.json 2>/dev/null; echo rep $rep rc=$?
done
timeout 900 python bench.py --steps 2000 --warmup 20 > gpurun_out/e2c_g1.json 2> gpurun_out/e2c_g1.err; echo g1 rc=$?
exit 0
