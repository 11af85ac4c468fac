#!/bin/bash
# A/B of library variants at G GPUs on one box: bash tools/ab_multi.sh G "variantA variantB" [bench args]
# (tools/variants/<name>.so; each run twice, interleaved). Prints value, BSP ms and ASP ms per variant.
G=$1; VARS=$2; shift 2
for i in 1 2; do for v in $VARS; do
  SS_LIB_VARIANT=tools/variants/$v.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $G --no-e2e --no-cpu-baseline \
    "$@" 2>/dev/null | tail -1 > /tmp/ab_line.json
  python - "$v" <<'PY'
import json, sys
d = json.load(open("/tmp/ab_line.json")); p = d["phases"]
print(f"{sys.argv[1]:10s} {d['value']:9.1f} steps/s  bsp {p['bsp_ms_per_step']*1e3:7.1f} us  asp {p['asp_ms_per_round']*1e3:7.1f} us  "
      + "  ".join(f"{k} {v['avg_us']:.1f}" for k, v in d["kernels"].items()))
PY
done; done
