# one GPU: producer warp + empty barriers in the streaming ring (cur) vs per-item CTA barrier (base = HEAD)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multi_gpu" > gpurun_out/prod_suite.log 2>&1; echo suite rc=$?; tail -1 gpurun_out/prod_suite.log
for rep in 1 2; do for V in cur base; do
if [ $V = base ]; then export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/base_head.so; else unset SS_LIB_VARIANT; fi
timeout 300 python bench.py --config 3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/prod_c3_${V}_$rep.json 2>/dev/null; echo c3 $V rc=$?
timeout 300 python bench.py --config 5a --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/prod_c5a_${V}_$rep.json 2>/dev/null; echo c5a $V rc=$?
done; done
exit 0
