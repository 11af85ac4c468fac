# one-GPU check of the current tree: single-GPU parity suite, bench configs 3 and 2, sanitizer cases
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_g1_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "not multi_gpu" > gpurun_out/r02_g1_suite.log 2>&1; echo suite rc=$?; tail -3 gpurun_out/r02_g1_suite.log
timeout 600 python bench.py --steps 2000 --warmup 20 > gpurun_out/r02_bench_c3_g1.json 2> gpurun_out/r02_bench_c3_g1.err; echo bench3 rc=$?
timeout 600 python bench.py --config 2 --steps 5000 --warmup 50 --no-cpu-baseline > gpurun_out/r02_bench_c2_g1.json 2> gpurun_out/r02_bench_c2_g1.err; echo bench2 rc=$?
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py > gpurun_out/r02_racecheck.log 2>&1; echo racecheck rc=$?; tail -4 gpurun_out/r02_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > gpurun_out/r02_synccheck.log 2>&1; echo synccheck rc=$?; tail -4 gpurun_out/r02_synccheck.log
