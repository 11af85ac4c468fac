#!/bin/bash
# One GPU: the GPU test suite, the default bench line, config 2, the ncu launch list and one ncu --set full capture
# of the two sync kernels (each ncu pass only after the same command exited 0 without ncu).
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config 2 --steps 3000 --warmup 50 > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; echo "c2 rc=$?"
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
$B > /dev/null 2>&1 && echo "B rc=0" && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv $B > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"asp_replay|bsp_update" -s 6 -c 2 -o gpurun_out/f_full $B > gpurun_out/f_ncu.log 2>&1; echo "ncu full rc=$?"
