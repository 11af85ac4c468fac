cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_g4_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r02_g4_suite.log 2>&1; echo rc=$? >> gpurun_out/r02_g4_suite.log
tail -3 gpurun_out/r02_g4_suite.log
timeout 600 python bench.py --gpus 4 --steps 200 --warmup 20 > gpurun_out/r02_bench_c3_g4.json 2> gpurun_out/r02_bench_c3_g4.err; echo bench4 rc=$?
timeout 600 python bench.py --gpus 2 --steps 200 --warmup 20 > gpurun_out/r02_bench_c3_g2.json 2> gpurun_out/r02_bench_c3_g2.err; echo bench2 rc=$?
head -c 600 gpurun_out/r02_bench_c3_g4.json
