# two GPUs: programmatic dependent launch on / off at G = 2 (configs 2 and 3), two passes
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for V in cur nopdl; do
if [ $V = nopdl ]; then export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/pdl_PDL1.so; else unset SS_LIB_VARIANT; fi
timeout 600 python bench.py --gpus 2 --config 2 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/pdl2_c2_${V}_$rep.json 2>/dev/null; echo c2 $V rc=$?
timeout 600 python bench.py --gpus 2 --config 3 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/pdl2_c3_${V}_$rep.json 2>/dev/null; echo c3 $V rc=$?
done; done
