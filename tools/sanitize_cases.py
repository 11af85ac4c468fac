"""Small single-GPU cases for compute-sanitizer (racecheck / synccheck / memcheck) on the hand-synchronised kernels:
the TMA window kernel in both instantiations (ring refilled under per-item CTA barriers; ring never reused, barrier-free),
windows with BSP supersteps, the scalar (unaligned) window kernel, and bsp_update (a superstep too large for a window).
Each case is also checked bit-exact against the oracle, so a sanitizer run doubles as a parity run.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as orc  # noqa: E402  (test infrastructure: this is a checking tool)
from paper_2104_08364_b200 import syncswitch as ss  # noqa: E402

SEED = 20241018


def dev(j, k, P, offset=0):
    buf = torch.empty(P + offset, device="cuda")
    out = buf[offset:]
    ss.ss_check(ss.ss_synth_grad(SEED, j, k, 0, P, out))
    return out


def case(name, P, n, S, pushes, bsp_steps, offset=0, window=16):
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    g.set_window(window)
    keep = []
    for t in range(bsp_steps):
        gs = [dev(j, t, P, offset) for j in range(n)]
        keep += gs
        g.bsp_step(gs)
        assert o.bsp_step([orc.synth_grad(SEED, j, t, 0, P) for j in range(n)]) == 0
    g.switch(ss.SS_ASP, 0)
    o.switch(orc.ASP, 0)
    dst = torch.empty(P, device="cuda")
    v = g.version
    for p in range(pushes):
        j = p % n
        gd = dev(j, 100 + p, P, offset)
        keep.append(gd)
        g.asp_push(j, gd, v)
        assert o.asp_push(j, orc.synth_grad(SEED, j, 100 + p, 0, P), v)[0] == 0
    g.pull(0, dst)
    snap = o.pull(0)[1]
    g.sync()
    assert np.array_equal(g.params(), o.params()) and np.array_equal(dst.cpu().numpy(), snap), name
    g.close()
    print(f"{name}: ok (P={P}, n={n}, pushes={pushes}, supersteps={bsp_steps}, offset={offset})", flush=True)


if __name__ == "__main__":
    torch.cuda.init()
    case("tma ring refilled (kRefill=true)", 300_007, 4, 4, 12, 0)
    case("tma ring never reused (kRefill=false)", 4099, 2, 2, 2, 0)
    case("window with BSP supersteps + pushes", 200_003, 4, 4, 6, 3)
    case("scalar window (unaligned sources)", 20_011, 3, 3, 5, 2, offset=1)
    case("bsp_update (superstep of 130 workers, outside the window)", 4099, 130, 2, 0, 1)
