#!/usr/bin/env python
"""Launch-gap probe for the fused multi-GPU path (torchrun, one process per GPU): times K bench steps (BSP + switch +
n push/pull + switch) of a config with per-kernel profiling events on or off; with SS_TRACE set, the per-launch
stamps (tools/trace_report.py) show where the device time goes.

    torchrun --nproc-per-node G tools/gap_probe.py --config 2 --steps 500 --prof 0
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, SEED  # noqa: E402
from paper_2104_08364_b200 import syncswitch as ss  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--prof", type=int, default=0)
    ap.add_argument("--fused", type=int, default=2)
    ap.add_argument("--graph", type=int, default=0, help="time replays of one captured step instead")
    a = ap.parse_args()
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[a.config]
    P, n, S = cfg["P"], cfg["n"], cfg["S"]
    hosted = [j for j in range(n) if (j * world) // n == rank]
    w0 = torch.zeros(P, device="cuda")
    g = ss.SyncSwitch(w0, S, n, 0.1, 0.9)
    if world > 1:
        uid = [ss.ss_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        g.init_dist(rank, world, uid[0])
        g.set_fused(a.fused)
    g.set_window(cfg["window"])
    ring = {(j, r): torch.empty(P, device="cuda") for j in hosted for r in range(2)}
    for (j, r), buf in ring.items():
        ss.ss_check(ss.ss_synth_grad(SEED, j, r, 0, P, buf))
    dst = {j: (g.pull_buffer(j) if world > 1 and a.fused else ss.ptr(torch.empty(P, device="cuda")))
           for j in hosted}
    gp = (ctypes.c_void_p * max(len(hosted), 1))(*[ss.ptr(ring[(j, 0)]) for j in hosted])
    ws = np.array(hosted, dtype=np.int32)
    vs = np.zeros(max(len(hosted), 1), dtype=np.int64)
    ev = (ss.ss_event * (2 * n))()
    for j in range(n):
        b = ring.get((j, 1))
        ev[2 * j] = ss.ss_event(0, j, 0, ss.ptr(b) if b is not None else None, None)
        ev[2 * j + 1] = ss.ss_event(1, j, 0, None, dst.get(j))
    L, c = ss.lib, g.ctx

    def step(ver):
        vs[:] = ver
        for j in range(n):
            ev[2 * j].version = ver + 1
        s = L.ss_bsp_step(c, ctypes.cast(gp, ctypes.c_void_p), ws.ctypes.data, vs.ctypes.data, len(hosted))
        s = s or L.ss_switch(c, ss.SS_ASP, 0)
        s = s or L.ss_asp_replay(c, ctypes.cast(ev, ctypes.c_void_p), 2 * n, None)
        s = s or L.ss_switch(c, ss.SS_BSP, 0)
        assert s == 0, g.last_error()
        return ver + 1 + n

    ver = 0
    for _ in range(20):
        ver = step(ver)
    g.profile(bool(a.prof))
    stream = torch.cuda.ExternalStream(g.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    import time
    if a.graph:
        g.capture_begin()
        ver = step(ver)
        g.capture_end()
        g.capture_replay(20)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    e0.record(stream)
    h0 = time.perf_counter()
    if a.graph:
        g.capture_replay(a.steps)
    else:
        for _ in range(a.steps):
            ver = step(ver)
    host_us = 1e6 * (time.perf_counter() - h0) / a.steps
    e1.record(stream)
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / a.steps
    t = torch.tensor([us], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"config {a.config} G={world} fused={a.fused} prof={a.prof} graph={a.graph}: {t.item():.2f} us/step "
              f"(host issue {host_us:.2f} us/step on rank 0)", flush=True)
    g.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
