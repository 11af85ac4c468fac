#!/usr/bin/env python
"""Tile / pipeline-depth sweep of the TMA replay kernel (asp_replay_tma_kernel).

    python tools/replay_sweep.py build            # here: builds tools/variants/lib_T<tile>_S<stages>.so
    python tools/replay_sweep.py run [--config 3] # on the GPU: bench.py per variant, prints asp_replay us and frac
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "variants")
VARIANTS = [(2048, 6), (2048, 10), (2048, 12), (2048, 14), (2048, 16), (2048, 24), (1024, 20), (4096, 6), (4096, 8), (4096, 12)]


def name(t, s):
    return os.path.join(OUT, f"lib_T{t}_S{s}.so")


def build():
    sys.path.insert(0, ROOT)
    from paper_2104_08364_b200.build import build as b
    os.makedirs(OUT, exist_ok=True)
    for t, s in VARIANTS:
        b(out=name(t, s), defines=(f"SS_TMA_TILE={t}", f"SS_TMA_STAGES={s}"))
        print("built", name(t, s), flush=True)


def run(config):
    for t, s in VARIANTS:
        env = dict(os.environ, SS_LIB_VARIANT=name(t, s))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", "1000",
                            "--no-e2e", "--no-cpu-baseline"], capture_output=True, text=True, env=env, timeout=300)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            k = d["kernels"]["asp_replay"]
            print(f"tile {t:5d} stages {s:2d}: {d['value']:9.1f} steps/s  asp_replay {k['avg_us']:8.2f} us "
                  f"frac {k['frac']:.4f}  bsp_update frac {d['kernels']['bsp_update']['frac']:.4f}", flush=True)
        except Exception:
            print(f"tile {t} stages {s}: failed\n{r.stderr[-1500:]}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "3")
