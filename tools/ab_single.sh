#!/bin/bash
# A/B of two library builds on one GPU, interleaved twice: bash tools/ab_single.sh "head new" <config> [steps]
VARS=$1; CFG=$2; STEPS=${3:-1000}
for i in 1 2; do for v in $VARS; do
  SS_LIB_VARIANT=tools/variants/$v.so timeout 300 python bench.py --config $CFG --steps $STEPS --no-e2e \
    --no-cpu-baseline 2>/dev/null > /tmp/ab_line.json
  python - "$v" <<'PY'
import json, sys
d = json.load(open("/tmp/ab_line.json")); k = d["kernels"]
print(f"{sys.argv[1]:6s} {d['value']:9.1f} steps/s  graph {d['graph'].get('steps_per_s', 0):9.1f}  " +
      "  ".join(f"{n} {v['avg_us']:.2f} us ({v['frac']:.4f})" for n, v in k.items()))
PY
done; done
