# one GPU: shared event table in the streaming form only (cur) vs HEAD (base): single-GPU suite, configs 2 and 3
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/sev2_suite.log 2>&1; echo suite rc=$?; tail -1 gpurun_out/sev2_suite.log
for rep in 1 2; do for V in cur base; do
if [ $V = base ]; then export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/base_head.so; else unset SS_LIB_VARIANT; fi
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/sev2_c2_${V}_$rep.json 2>/dev/null; echo c2 $V rc=$?
timeout 300 python bench.py --config 3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/sev2_c3_${V}_$rep.json 2>/dev/null; echo c3 $V rc=$?
done; done
exit 0
