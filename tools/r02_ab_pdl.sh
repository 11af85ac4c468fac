# one GPU: programmatic dependent launch on/off (and the round-1 kernels) on configs 4, 2 and 3
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for V in cur nopdl r01; do
case $V in cur) unset SS_LIB_VARIANT;; nopdl) export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/pdl_PDL1.so;; r01) export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/r01_kernels.so;; esac
timeout 300 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/ab_c4_${V}_$rep.json 2>/dev/null; echo c4 $V rc=$?
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/ab_c2_${V}_$rep.json 2>/dev/null; echo c2 $V rc=$?
done; done
unset SS_LIB_VARIANT
