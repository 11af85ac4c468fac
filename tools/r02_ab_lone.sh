# one GPU: lone superstep through bsp_update (default) vs the window kernel, config 2 and config 3, two passes
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for V in cur lone; do
if [ $V = lone ]; then export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/lone_WINDOW1.so; else unset SS_LIB_VARIANT; fi
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/lone_c2_${V}_$rep.json 2>/dev/null; echo c2 $V rc=$?
done; done
exit 0
