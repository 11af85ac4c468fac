#!/bin/bash
# Last round-1 check on one GPU: smoke, the GPU suite, and an ncu capture of config 2's two sync kernels (warm L2 as
# the bench runs them: --cache-control none).
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/z_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --config 2 --steps 30 --warmup 25 --no-e2e --no-cpu-baseline"
$B > /dev/null 2>&1 && echo "B rc=0" && \
timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"asp_replay|bsp_update" \
  -s 60 -c 2 -o gpurun_out/z_c2_full $B > gpurun_out/z_ncu.log 2>&1; echo "ncu rc=$?"
