# two GPUs: e2e (host buffers) variance check of the config-3 line
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
timeout 600 python bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2e_g2_$rep.json 2>/dev/null; echo rep $rep rc=$?
done
python tools/pcie_probe.py > gpurun_out/e2e_pcie_probe.txt 2>&1; echo probe rc=$?
exit 0
