# one GPU: window events in shared memory (cur) vs kernel-parameter reads (base = HEAD), configs 2 and 3, interleaved
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/sev_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/sev_parity.log
for rep in 1 2 3; do for V in cur base; do
if [ $V = base ]; then export SS_LIB_VARIANT=$GRAFT_REPO_ROOT/tools/variants/base_head.so; else unset SS_LIB_VARIANT; fi
timeout 300 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/sev_c2_${V}_$rep.json 2>/dev/null; echo c2 $V rc=$?
[ $rep -le 2 ] && timeout 300 python bench.py --config 3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/sev_c3_${V}_$rep.json 2>/dev/null
done; done
