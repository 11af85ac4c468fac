#!/usr/bin/env python
"""Compile-time tuning sweeps of the single-GPU kernels (variants of the whole library built with -D knobs).

    python tools/kernel_sweep.py build <set>            # here: tools/variants/<set>_<tag>.so
    python tools/kernel_sweep.py run <set> [--config 3] # on the GPU: bench.py per variant
Sets: replay (asp_replay_tma_kernel tile x stages; profiles/r01_replay_sweep.txt, r02_replay_sweep.txt), bsp (bsp_update
float4 per thread x gradients loaded together), pdl (programmatic dependent launch off; profiles/r02_pdl_ab.txt).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "variants")
SETS = {
    "replay": [{"SS_TMA_TILE": t, "SS_TMA_STAGES": s} for t, s in
               [(2048, 6), (2048, 10), (2048, 12), (2048, 14), (2048, 16), (1024, 20), (4096, 6)]],
    "bsp": [{"SS_BSP_U": u, "SS_BSP_G": g} for u, g in [(2, 8), (1, 8), (1, 4), (2, 4), (4, 4), (4, 2), (3, 8)]],
    "pdl": [{"SS_NO_PDL": 1}],   # programmatic dependent launch off (A/B against the default library)
}


def tag(d):
    return "_".join(f"{k.split('_')[-1]}{v}" for k, v in d.items())


def variants(name):
    """Distinct variants of a set (a set may list one twice to interleave repeated runs on the same box)."""
    out = []
    for d in SETS[name]:
        if d not in out:
            out.append(d)
    return out


def path(name, d):
    return os.path.join(OUT, f"{name}_{tag(d)}.so")


def build(name):
    sys.path.insert(0, ROOT)
    from paper_2104_08364_b200.build import build as b
    os.makedirs(OUT, exist_ok=True)
    for d in variants(name):
        b(out=path(name, d), defines=[f"{k}={v}" for k, v in d.items()])
        print("built", path(name, d), flush=True)


def run(name, config):
    for d in SETS[name]:
        env = dict(os.environ, SS_LIB_VARIANT=path(name, d))
        steps = "1000" if config not in ("2",) else "3000"
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", steps,
                            "--no-e2e", "--no-cpu-baseline"], capture_output=True, text=True, env=env, timeout=300)
        try:
            line = json.loads(r.stdout.strip().splitlines()[-1])
            k = line["kernels"]
            print(f"{tag(d):18s} {line['value']:9.1f} steps/s  bsp_update {k['bsp_update']['avg_us']:8.2f} us "
                  f"frac {k['bsp_update']['frac']:.4f}  asp_replay {k['asp_replay']['avg_us']:8.2f} us "
                  f"frac {k['asp_replay']['frac']:.4f}", flush=True)
        except Exception:
            print(f"{tag(d)}: failed\n{r.stderr[-1500:]}", flush=True)


if __name__ == "__main__":
    cmd, name = sys.argv[1], sys.argv[2]
    if cmd == "build":
        build(name)
    else:
        run(name, sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "3")
