#!/usr/bin/env python
"""Benchmark of the Sync-Switch synchronization path on B200 (BASELINE.json metric: BSP sync steps/s and ASP pushes/s
at 1/2/4/8 B200; HBM & NVLink GB/s vs peak).

One bench STEP is one pass of the whole hot path over one batch of synthetic gradients:
  BSP superstep (n gradients: barrier, aggregate, momentum update, broadcast)  -> in-place switch to ASP
  -> one ASP round (n pushes, each followed by the pusher's pull; staleness 0..n-1) -> in-place switch back to BSP.
Workload at N=1 and by default: BASELINE config 3 (ResNet-50-shaped, P = 25,557,032 fp32, n = S = 8). Gradients
come from the seeded synth_grad kernel into per-worker rings before timing: 2 slots (BSP, ASP) per set, R sets
rotated step by step with R chosen so that R steps' gradients are >= 3x the 126 MB L2 (R = 1 at config 3, whose step
streams ~3.3 GB), so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|2|5a..5d] [--impl ours|reference]
N > 1: one process per GPU — under torchrun, or started by bench.py itself (torch.distributed.run on 127.0.0.1)
when WORLD_SIZE is unset; the fused peer-memory exchange over NVLink (scatter -> owner update + broadcast for BSP,
owner-routed pushes and pulls for ASP), NCCL for set-up and agreement; strong scaling (P and n fixed).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "3": dict(P=25_557_032, n=8, S=8, window=16, name="config3: ResNet-50-shaped sync, P=25,557,032 fp32, "
                                                        "n=8 workers, S=8 shards"),
    "2": dict(P=464_154, n=8, S=8, window=16, name="config2: ResNet-32/CIFAR-10-shaped sync, P=464,154 fp32, "
                                                     "n=8 workers, S=8 shards"),
    "5a": dict(P=100_000_000, n=8, S=8, window=16, name="config5: large-model sync, P=1e8 fp32, n=S=8"),
    "5b": dict(P=250_000_000, n=8, S=8, window=16, name="config5: large-model sync, P=2.5e8 fp32, n=S=8"),
    "5c": dict(P=500_000_000, n=8, S=8, window=16, name="config5: large-model sync, P=5e8 fp32, n=S=8"),
    "5d": dict(P=1_000_000_000, n=8, S=8, window=16, name="config5: large-model sync, P=1e9 fp32, n=S=8"),
    "1": dict(P=8192, n=2, S=2, window=1, name="config1: toy softmax regression (d=1024 incl. bias, C=8, P=8,192), "
              "2 workers, 2 shards, 1,000 points, W=100 B, switch BSP->ASP at 50% (25 BSP steps + 50 ASP pushes)"),
    "4": dict(P=25_557_032, n=8, S=8, window=16, name="config4: ASP straggler scenario, worker 7 4x slow for "
              "100,000 ticks during BSP, greedy switching (P:1421), P=25,557,032, n=S=8"),
}
SCENARIO4 = dict(n_workers=8, batch=128, total_samples=64000 * 128, quota_num=1, quota_den=4, period=1000, jitter=0,
                 sched_seed=7, grad_seed=20241018, slow_worker=7, slow_factor=4, slow_t0=20000, slow_t1=120000,
                 window_ticks=10000, K=3)
L2_BYTES = 126 * 1024 * 1024
# ss_kernel_stats ids: 4 = the window kernel applying a BSP superstep together with the ASP events queued behind it
# (one GPU: the superstep joins the window, see ss_bsp_step)
KERNEL_NAMES = ["bsp_update", "asp_replay", "local_sum", "scatter", "bsp_window"]
METRIC = "BSP sync steps/s and ASP pushes/s at 1/2/4/8 B200; HBM & NVLink GB/s vs peak"
UNIT = "steps/s (1 step = 1 BSP superstep + switch + n ASP push/pull + switch)"
SEED = 20241018
PROF_NOTE = ("CUDA events around every launch on the library stream, in a second pass of the same K steps right "
             "after the uninstrumented timed region")


# The JSON line is the only thing bench.py writes to stdout: native libraries (NCCL prints its version banner from
# the communicator set-up inside the library) write to file descriptor 1 directly, so fd 1 is pointed at stderr for
# the whole run and the line goes to a private copy of the original stdout.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(line: dict):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="3", choices=sorted(CONFIGS))
    ap.add_argument("--scenario-samples", type=int, default=16000 * 128,
                    help="config 4: total samples W of the scenario (the paper's 64K x 128 takes minutes)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fused", default="auto", choices=["auto", "0", "1", "2", "3"],
                    help="G>1 exchange: 0 NCCL, 1 fused exact, 2 fused pre-summed, 3 fused pull; auto = 3 if n <= G else 2")
    ap.add_argument("--workload", action="store_true",
                    help="config 2/3: sync-only time of the whole 64K-iteration workload, pure BSP / pure ASP / "
                         "switched (Table I remap)")
    ap.add_argument("--window", type=int, default=0, help="ASP replay window in events (0: the config's default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def step_floor(world: int, P: int, S: int, n: int, steps_per_s: float, hbm_peak: float) -> dict:
    """The bench step's floor on this N: the bytes the method must move through the bounding link, at its peak.
    G > 1: per GPU per direction, the BSP exchange (RS + AG: 2(G-1)/G * 4 P_pad) plus the ASP round (n pushes routed
    to the owners and n pull snapshots routed back, n/G of each per GPU: 2 (n/G)(G-1)/G * 4 P_pad), over 900 GB/s
    NVLink; G = 1: the two kernels' HBM bytes ((n + 4) 4P for the superstep, (2n + 4) 4P for the ASP round) over the
    measured copy rate."""
    if world > 1:
        P_pad = S * (((P + S - 1) // S + 31) // 32 * 32)
        nv_bytes = 2 * (world - 1) / world * 4 * P_pad * (1 + n / world)
        floor = {"bound": "nvlink", "bytes_per_gpu_per_direction": nv_bytes, "peak_GBps": 900.0,
                 "steps_per_s_at_peak": 900e9 / nv_bytes}
    else:
        step_bytes = (3 * n + 8) * 4 * P
        floor = {"bound": "hbm", "bytes": step_bytes, "peak_GBps": hbm_peak,
                 "steps_per_s_at_peak": hbm_peak * 1e9 / step_bytes}
    floor["frac_of_floor"] = steps_per_s / floor["steps_per_s_at_peak"]
    return floor


def ncu_traffic(kernel: str, config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config, {}).get(kernel)
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2104_08364_b200 import syncswitch as ss

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = dict(CONFIGS[args.config])
    if args.config.startswith("5") and world > 1:
        # n = S = G at G in {2, 4, 8} (one worker and one shard per GPU); n = S = 8 at G = 1
        cfg.update(n=world, S=world, name=cfg["name"].replace("n=S=8", f"n=S=G={world}"))
    P, n, S, win = cfg["P"], cfg["n"], cfg["S"], args.window or cfg["window"]
    hosted = [j for j in range(n) if (j * world) // n == rank]

    # initial parameters (seeded, identical on every rank) and the context
    w0 = torch.empty(P, device="cuda")
    ss.ss_check(ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0))
    w0.mul_(64.0)
    torch.cuda.synchronize()
    g = ss.SyncSwitch(w0, S, n, 0.1, 0.9)
    if world > 1:
        uid = [ss.ss_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        g.init_dist(rank, world, uid[0])
    # exchange: one worker per GPU or fewer (the paper's layout) -> the one-kernel pull exchange (mode 3); more workers
    # than GPUs -> each rank pre-sums its workers and scatters one slice per owner (mode 2)
    fused = (3 if n <= world else 2) if args.fused == "auto" else int(args.fused)
    if world > 1:
        g.set_fused(fused)
    g.set_window(win)
    del w0

    # gradient rings: R sets of 2 slots per hosted worker (slot 2q feeds set q's BSP superstep, slot 2q+1 its ASP
    # round); step k uses set k mod R. R is chosen so that the gradients one rank reads over R consecutive steps are
    # >= 3x the 126 MB L2: every step's inputs were last touched >= R-1 steps (>= 2 L2 capacities of traffic) earlier,
    # so small models are timed with their gradients streamed from HBM, not replayed out of L2. The PS state (w, v)
    # and the pull buffers are the library's and stay where the hardware keeps them.
    set_bytes = 2 * max(len(hosted), 1) * 4 * P
    R = max(1, math.ceil(3 * L2_BYTES / set_bytes))
    ring = {(j, r): torch.empty(P, device="cuda") for j in hosted for r in range(2 * R)}
    if world > 1 and fused == 3 and R == 1:
        # mode 3 reads superstep gradients in place from the exported gradient buffers: the worker writes its
        # gradient there (zero copy). With R > 1 sets the sets stay separate buffers, copied in per superstep.
        for j in hosted:
            ring[(j, 0)] = g.grad_buffer(j)
    for (j, r), buf in ring.items():
        ss.ss_check(ss.ss_synth_grad(SEED, j, r % 2, 0, P, buf))   # every set holds the same values (k = 0, 1)
    if world > 1 and fused:
        pull_dst = {j: g.pull_buffer(j) for j in hosted}     # zero-copy pulls into the NVLink-mapped buffers
    else:
        pull_dst = {j: torch.empty(P, device="cuda") for j in hosted}
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(g.stream)

    class Step:
        """One bench step through the C-ABI with prebuilt argument arrays: ss_bsp_step, ss_flush, ss_switch(ASP),
        ss_asp_replay(n pushes, each followed by its pull), ss_flush, ss_switch(BSP). The flushes stand for the
        data dependencies of real training — the workers compute their first ASP gradients from the parameters after
        the superstep, and the next superstep's gradients from the parameters after the ASP round — so the library's
        window batching never fuses work across them (one GPU: one kernel for the superstep, one for the ASP round).
        `mark` (optional) is recorded on the library's stream between the BSP and the ASP phase."""

        def __init__(self, grad_src, dst_src):
            import ctypes
            self.ct = ctypes
            self.k = len(hosted)
            self.gp = (ctypes.c_void_p * max(self.k, 1))(*[ss.ptr(grad_src[(j, 0)]) for j in hosted])
            self.ws = np.array(hosted, dtype=np.int32)
            self.vs = np.zeros(max(self.k, 1), dtype=np.int64)
            self.ev = (ss.ss_event * (2 * n))()
            for j in range(n):
                self.ev[2 * j] = ss.ss_event(0, j, 0, ss.ptr(grad_src.get((j, 1))), None)
                self.ev[2 * j + 1] = ss.ss_event(1, j, 0, None, ss.ptr(dst_src.get(j)))
            self.gp_c = ctypes.cast(self.gp, ctypes.c_void_p)
            self.ev_c = ctypes.cast(self.ev, ctypes.c_void_p)

        def __call__(self, ver, mark=None):
            L, c = ss.lib, g.ctx
            self.vs[:] = ver
            for j in range(n):
                self.ev[2 * j].version = ver + 1
            s = L.ss_bsp_step(c, self.gp_c, self.ws.ctypes.data, self.vs.ctypes.data, self.k)
            s = s or L.ss_flush(c)
            if mark is not None:
                mark.record(stream)
            s = s or L.ss_switch(c, ss.SS_ASP, 0)
            s = s or L.ss_asp_replay(c, self.ev_c, 2 * n, None)
            s = s or L.ss_flush(c)
            s = s or L.ss_switch(c, ss.SS_BSP, 0)
            if s:
                raise ss.SSError(s, g.last_error())
            return ver + 1 + n

        def bsp_only(self, ver):
            """One BSP superstep (under BSP)."""
            self.vs[:] = ver
            s = ss.lib.ss_bsp_step(g.ctx, self.gp_c, self.ws.ctypes.data, self.vs.ctypes.data, self.k)
            s = s or ss.lib.ss_flush(g.ctx)       # the next superstep's gradients depend on this one
            if s:
                raise ss.SSError(s, g.last_error())
            return ver + 1

        def asp_window(self, ver, first):
            """One ASP window under ASP: n pushes, each followed by the pusher's pull. Push j sends the version of
            its last pull: the switch's version for the first window (a BSP superstep sets every base), afterwards
            ver - n + j + 1 (staleness n - 1)."""
            for j in range(n):
                self.ev[2 * j].version = ver if first else ver - n + j + 1
            s = ss.lib.ss_asp_replay(g.ctx, self.ev_c, 2 * n, None)
            s = s or ss.lib.ss_flush(g.ctx)       # each worker's next push depends on its pull
            if s:
                raise ss.SSError(s, g.last_error())
            return ver + n

    steps_dev = [Step({(j, r): ring[(j, 2 * q + r)] for j in hosted for r in range(2)}, pull_dst) for q in range(R)]
    n_call = [0]

    def step_dev(ver, mark=None):
        st = steps_dev[n_call[0] % R]
        n_call[0] += 1
        return st(ver, mark)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ver = g.version
    for _ in range(args.warmup):
        ver = step_dev(ver)
    barrier()

    # Timed region: K steps, no instrumentation between the kernels (per-launch timing events cost device time: at
    # G = 2 on config 2 they stretch a step from 67 to 117 us, tools/gap_probe.py) -> value, ms_per_step.
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    e_start, e_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e_start.record(stream)
    for k in range(args.steps):
        ver = step_dev(ver)
    e_stop.record(stream)
    barrier()
    total_ms = e_start.elapsed_time(e_stop)
    # Profiled pass of the same K steps right after it: CUDA events around every launch on the library's stream
    # (ss_profile) and at the phase boundaries -> kernels, roofline, phases.
    g.profile(True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    barrier()
    ev[0].record(stream)
    for k in range(args.steps):
        ver = step_dev(ver, mark=ev[2 * k + 1])
        ev[2 * k + 2].record(stream)
    barrier()
    clk = clocks.stop()
    prof_ms = ev[0].elapsed_time(ev[-1])
    bsp_ms = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps))
    asp_ms = sum(ev[2 * k + 1].elapsed_time(ev[2 * k + 2]) for k in range(args.steps))
    kst = {name: g.kernel_stats(i) for i, name in enumerate(KERNEL_NAMES)}
    g.profile(False)
    t = torch.tensor([total_ms, bsp_ms, asp_ms, prof_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, bsp_ms, asp_ms, prof_ms = t.tolist()
    launches = sum(k["launches"] for k in kst.values())

    # Pure-protocol rates (the metric's "BSP sync steps/s" and "ASP pushes/s" as a training phase runs them):
    # supersteps back to back, then ASP windows back to back, each run timed by two events on the library's stream
    # with no per-launch instrumentation (max over ranks).
    nr = max(20, args.steps // 2)
    ver = g.version
    pe = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    barrier()
    pe[0].record(stream)
    for t in range(nr):
        ver = steps_dev[t % R].bsp_only(ver)
    pe[1].record(stream)
    barrier()
    g.switch(ss.SS_ASP, 0)
    barrier()
    pe[2].record(stream)
    for t in range(nr):
        ver = steps_dev[t % R].asp_window(ver, t == 0)
    g.sync()
    pe[3].record(stream)
    barrier()
    g.switch(ss.SS_BSP, 0)
    pt = torch.tensor([pe[0].elapsed_time(pe[1]), pe[2].elapsed_time(pe[3])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    bsp_only_ms, asp_only_ms = pt.tolist()
    rates = {"bsp_steps_per_s": nr / (bsp_only_ms / 1e3), "bsp_us_per_step": 1e3 * bsp_only_ms / nr,
             "asp_pushes_per_s": n * nr / (asp_only_ms / 1e3), "asp_us_per_window": 1e3 * asp_only_ms / nr,
             "supersteps": nr, "windows": nr, "pushes_per_window": n,
             "note": "pure BSP supersteps back to back, then pure ASP windows (n pushes, each followed by its pull) "
                     "back to back; two CUDA events per run, no per-launch instrumentation; max over ranks. Every "
                     "superstep and every window is flushed (issued as its own kernel), as the data dependencies of "
                     "real training force"}
    ver = g.version
    st = g.stats(64)
    assert st["status"] == 0 and g.sync_status() == 0, g.last_error()

    # the same step replayed from a CUDA graph (ss_capture_*; every rank captures and replays it): host launch
    # overhead removed. Informational (single GPU: faster for latency-bound configs; G > 1: the replayed fused kernels
    # run slower than the eager ones, profiles/r01_summary.md), so a failure here does not cost the line.
    graph = None
    try:
        g.capture_begin()
        for _ in range(R):            # one step per gradient set: the replay streams the same inputs as eager
            ver = step_dev(ver)
        g.capture_end()
        g.capture_replay(max(1, args.warmup // R))
        reps = max(1, args.steps // R)
        ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ge0.record(stream)
        g.capture_replay(reps)
        ge1.record(stream)
        barrier()
        gt = torch.tensor([ge0.elapsed_time(ge1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gms = gt.item()
        assert g.sync_status() == 0, g.last_error()
        graph = {"steps_per_s": round(reps * R / (gms / 1e3), 3), "ms_per_step": gms / (reps * R),
                 "steps": reps * R,
                 "note": f"ss_capture_replay: {R} captured step(s) (one per gradient set) replayed on every rank; "
                         "host protocol state advanced identically"}
    except Exception as exc:          # noqa: BLE001 — reported, not fatal
        graph = {"error": str(exc)[:200]}
        try:
            g.capture_end()           # leave capture mode if the failure happened inside it
        except Exception:             # noqa: BLE001
            pass
    ver = g.version

    # e2e: same steps through the C-ABI with HOST (pinned) buffers, H2D / D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        hring = {(j, r): torch.empty(P, pin_memory=True) for j in hosted for r in range(2)}
        tmpd = torch.empty(P, device="cuda")
        for (j, r), buf in hring.items():          # the same values as the device ring (k = 0: BSP, k = 1: ASP)
            ss.ss_check(ss.ss_synth_grad(SEED, j, r, 0, P, tmpd))
            torch.cuda.synchronize()
            buf.copy_(tmpd)
        del tmpd
        hdst = {j: torch.empty(P, pin_memory=True) for j in hosted}
        del ring
        torch.cuda.empty_cache()
        if world == 1:
            # host data: flush each push with its pull so that a pull's D2H (copy_out stream) overlaps the next
            # push's H2D (copy_in stream); results are identical for any window size
            g.set_window(2)
        step_host = Step(hring, hdst)
        # warm-up: the library's staging ring for host buffers grows lazily to its full size (cudaMalloc of 4P-byte
        # slots); run enough untimed steps to fill it so no allocation falls inside the timed region
        for _ in range(max(args.e2e_steps, 16)):
            ver = step_host(ver)
            g.sync()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            ver = step_host(ver)
            g.sync()                   # the step's results (pull snapshots) are on the host
        e1.record(stream)
        barrier()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        h2d = 4 * P * 2 * n          # whole job: every worker's BSP and ASP gradient crosses PCIe once per step
        d2h = 4 * P * n              # and every worker's pull snapshot comes back
        e2e = {"value": args.e2e_steps / (et.item() / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "note": "pinned host gradients and pull destinations, copies staged by the library"}

    hbm_peak, peak_src = peaks()
    nvl_peak = 770.0   # measured NVLink peer copy per direction per GPU (B200_PROFILING.md; 900 nominal)
    # dominant kernel by device time among the path's kernels
    dom = max((k for k in kst if kst[k]["launches"]), key=lambda k: kst[k]["ms"])
    d = kst[dom]
    per_launch_s = d["ms"] / d["launches"] / 1e3
    if world > 1 and d["nvlink_bytes"] > 0:
        # fused multi-GPU path: the kernel is bound by what it must send over NVLink
        achieved = d["nvlink_bytes"] / d["launches"] / per_launch_s / 1e9
        roofline = {"bound": "nvlink", "kernel": dom, "achieved": round(achieved, 1), "peak": nvl_peak,
                    "unit": "GB/s", "frac": round(achieved / nvl_peak, 4), "traffic": None,
                    "bytes_per_launch": d["nvlink_bytes"] / d["launches"], "avg_launch_us": 1e6 * per_launch_s,
                    "peak_source": "measured NVLink peer copy 770 GB/s per direction (B200_PROFILING.md)",
                    "frac_of_nominal_900GBps": round(achieved / 900.0, 4),
                    # every GPU sending to every peer at once: SM-driven stores reach ~690 GB/s per GPU
                    # (tools/p2p_bench.cu, profiles/r01_p2p_alltoall_microbench.txt)
                    "frac_of_alltoall_sm_ceiling_690GBps": round(achieved / 690.0, 4),
                    "hbm_GBps": round(d["bytes"] / d["launches"] / per_launch_s / 1e9, 1), "measured_in": PROF_NOTE}
    else:
        achieved = d["bytes"] / d["launches"] / per_launch_s / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(achieved / hbm_peak, 4), "traffic": ncu_traffic(dom, args.config),
                    "bytes_per_launch": d["bytes"] / d["launches"], "avg_launch_us": 1e6 * per_launch_s,
                    "peak_source": peak_src, "frac_of_nominal_8TBps": round(achieved / 8000.0, 4),
                    "measured_in": PROF_NOTE}
    kernels = {}
    for name, k in kst.items():
        if k["launches"]:
            sec = k["ms"] / 1e3
            gbs = k["bytes"] / sec / 1e9
            kernels[name] = {"launches": k["launches"], "avg_us": round(1e3 * k["ms"] / k["launches"], 2),
                             "GBps": round(gbs, 1), "frac": round(gbs / hbm_peak, 4),
                             "share_of_step": round(k["ms"] / prof_ms, 4)}
            if k["nvlink_bytes"] > 0:
                kernels[name]["nvlink_GBps"] = round(k["nvlink_bytes"] / sec / 1e9, 1)
                kernels[name]["nvlink_frac_of_770"] = round(k["nvlink_bytes"] / sec / 1e9 / nvl_peak, 4)

    steps_per_s = args.steps / (total_ms / 1e3)
    # 1-GPU form: n BSP + n ASP gradients read, n pulls written, w and v read and written by each of the two kernels
    step_bytes = (3 * n + 8) * 4 * P / world
    if world == 1:
        phases = {"bsp_steps_per_s": args.steps / (bsp_ms / 1e3), "asp_pushes_per_s": n * args.steps / (asp_ms / 1e3),
                  "bsp_ms_per_step": bsp_ms / args.steps, "asp_ms_per_round": asp_ms / args.steps,
                  "profiled_ms_per_step": prof_ms / args.steps,
                  "note": "from the profiled pass (events at every launch and phase boundary); one GPU: the superstep "
                          "runs in bsp_update, the ASP round in the window kernel asp_replay"}
    else:
        phases = {"bsp_steps_per_s": args.steps / (bsp_ms / 1e3), "asp_pushes_per_s": n * args.steps / (asp_ms / 1e3),
                  "bsp_ms_per_step": bsp_ms / args.steps, "asp_ms_per_round": asp_ms / args.steps,
                  "note": "from the profiled pass (events at every launch and phase boundary)",
                  "profiled_ms_per_step": prof_ms / args.steps}
    if world > 1:
        # NCCL bus bandwidth convention for the BSP exchange: RS + AG each move (G-1)/G * 4 P_pad per GPU
        P_pad = S * (((P + S - 1) // S + 31) // 32 * 32)
        per_dir = 2 * (world - 1) / world * 4 * P_pad
        phases["bsp_nvlink_busbw_GBps"] = per_dir / (bsp_ms / args.steps / 1e3) / 1e9
        phases["bsp_nvlink_frac_of_900"] = phases["bsp_nvlink_busbw_GBps"] / 900.0
        phases["bsp_nvlink_frac_of_770_measured"] = phases["bsp_nvlink_busbw_GBps"] / 770.0
        rates["bsp_nvlink_busbw_GBps"] = per_dir / (bsp_only_ms / nr / 1e3) / 1e9
        rates["bsp_nvlink_frac_of_900"] = rates["bsp_nvlink_busbw_GBps"] / 900.0
    floor = step_floor(world, P, S, n, steps_per_s, hbm_peak)
    line = {
        "metric": METRIC, "value": round(steps_per_s, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded counter-hash gradients)",
        "config": {"workload": cfg["name"], "P": P, "n_workers": n, "n_shards": S, "asp_window_events": win,
                   "parallelism": f"sharded PS over {world} GPU(s)",
                   "exchange": "single GPU" if world == 1 else
                   ["NCCL RS/AG + send/recv", "fused peer-memory, exact", "fused peer-memory, pre-summed",
                    "fused one-kernel pull (gradient buffers read in place over NVLink)"][fused],
                   "gradient_sets": R,
                   "l2": (f"inputs larger than L2: {step_bytes / 1e9:.2f} GB streamed per step vs 126 MB L2, no flush"
                          if R == 1 else
                          f"inputs larger than L2: gradients rotate over {R} sets ({R * set_bytes / 1e6:.0f} MB per "
                          f"rank, >= 3x the 126 MB L2), no flush; PS state w, v ({8 * P / world / 1e6:.1f} MB) and "
                          f"pull buffers stay resident")},
        "phases": phases, "protocol_rates": rates, "step_floor": floor, "roofline": roofline, "kernels": kernels, "gpu_launches": launches, "clocks": clk,
        "graph": graph,
        "e2e": e2e,
        "protocol_check": {"version": st["version"], "hist_0_to_n": [int(x) for x in st["hist"][:n + 1]]},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        del g
        torch.cuda.empty_cache()
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
    g = None
    if rank == 0:
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------------------------------
def run_scenario(args):
    """Config 4: the online straggler scenario (ss_scenario_run) on 1 GPU; device time by CUDA events around the run.
    Reports protocol updates/s (BSP steps + ASP pushes per second, gradients generated in-line by synth_grad as the
    worker stand-in), the switch log, the staleness histogram and the dropped pushes."""
    import torch
    from paper_2104_08364_b200 import syncswitch as ss
    cfg = CONFIGS["4"]
    P, n, S = cfg["P"], cfg["n"], cfg["S"]
    sc = dict(SCENARIO4, total_samples=args.scenario_samples)
    w0 = torch.empty(P, device="cuda")
    ss.ss_check(ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0))
    w0.mul_(64.0)
    torch.cuda.synchronize()
    # warm-up: one short run of the same scenario on a throwaway context (kernel modules load lazily on first launch,
    # the scenario's buffers are allocated once by the allocator), then the timed run on a fresh context
    warm = ss.SyncSwitch(w0, S, n, 0.1, 0.9)
    warm.set_window(cfg["window"])
    s_w, _, _ = ss.ss_scenario_run(warm.ctx, dict(sc, total_samples=min(sc["total_samples"], 512 * 128)))
    assert s_w == 0, warm.last_error()
    warm.sync()
    warm.close()
    torch.cuda.synchronize()
    g = ss.SyncSwitch(w0, S, n, 0.1, 0.9)
    g.set_window(cfg["window"])
    stream = torch.cuda.ExternalStream(g.stream)
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    s, log, res = ss.ss_scenario_run(g.ctx, sc)
    e1.record(stream)
    g.sync()
    clk = clocks.stop()
    assert s == 0, g.last_error()
    ms = e0.elapsed_time(e1)
    st = g.stats(64)
    updates = res["bsp_steps"] + res["asp_pushes"]
    line = {"metric": METRIC, "value": round(updates / (ms / 1e3), 1),
            "unit": "protocol updates/s (BSP steps + ASP pushes, scenario incl. in-line gradient generation)",
            "n_gpus": 1, "steps": updates, "warmup": 1, "ms_per_step": ms / updates, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded counter-hash gradients)",
            "config": {"workload": cfg["name"], "P": P, "n_workers": n, "n_shards": S, "scenario": sc},
            "scenario": {"switches": [dict(zip(("tick", "version", "to", "reason"), e)) for e in log], **res,
                         "staleness_hist": {str(i): int(x) for i, x in enumerate(st["hist"]) if x}},
            "clocks": clk}
    emit(line)


# ------------------------------------------------------------------------------------------------------------------
def run_toy(args):
    """Config 1 (BASELINE configs[0]): the toy model trained through the library on 1 GPU — every update's gradient
    comes from the hand-written softmax_grad kernel on the worker's own pull (window 1: each pull is written before
    the gradient kernel reads it, all on the library's stream, no host synchronisation inside a run). W = 100 B
    samples switched at s = 0.5 (Table I: 25 BSP supersteps + 50 ASP pushes), seeded jittered schedule. A step = one
    whole training run from w = 0; value = protocol updates/s including the gradient kernels."""
    import ctypes

    import numpy as np
    import torch

    from inputs import TOY_RECIPE, minibatch_order, toy_split
    from paper_2104_08364_b200 import syncswitch as ss
    cfg = CONFIGS["1"]
    n, S, B, d, C = cfg["n"], cfg["S"], 16, 1024, 8
    P = d * C
    X, y, Xte, yte = toy_split()               # overlapping classes: still training at the switch (eta 0.1, mu 0.9)
    s_, (bsp_steps, asp_pushes, _) = ss.ss_table1(100 * B, B, n, 1, 2, [])
    ss.ss_check(s_)
    order = minibatch_order(1, len(X), n * bsp_steps + asp_pushes, B)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    Xb = [Xd[torch.from_numpy(order[b]).cuda()].contiguous() for b in range(len(order))]   # input pipeline
    yb = [yd[torch.from_numpy(order[b]).cuda()].contiguous() for b in range(len(order))]
    s_, (kind, worker, _) = ss.ss_schedule(n, [1000] * n, asp_pushes, jitter=100, seed=7)
    ss.ss_check(s_)
    losses = torch.zeros(bsp_steps * n + asp_pushes, device="cuda")
    grads = [torch.empty(P, device="cuda") for _ in range(max(n, 1))]
    snap = {j: torch.empty(P, device="cuda") for j in range(n)}
    L = ss.lib

    def one_run():
        g = ss.SyncSwitch(torch.zeros(P, device="cuda"), S, n, 0.1, 0.9)
        g.set_window(1)
        g.switch(ss.SS_ASP, bsp_steps)
        st = g.stream
        mb, li = 0, 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.ExternalStream(st)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(bsp_steps):
            g.pull(0, snap[0])
            for j in range(n):
                ss.ss_check(L.ss_softmax_grad(ss.ptr(Xb[mb]), ss.ptr(yb[mb]), B, d, C, ss.ptr(snap[0]),
                                              ss.ptr(grads[j]), losses.data_ptr() + 4 * li, ctypes.c_void_p(st)))
                mb, li = mb + 1, li + 1
            g.bsp_step(grads[:n])
        base = {}
        for kd, j in zip(kind, worker):
            j = int(j)
            if kd == 1:
                base[j] = g.pull(j, snap[j])
            else:
                ss.ss_check(L.ss_softmax_grad(ss.ptr(Xb[mb]), ss.ptr(yb[mb]), B, d, C, ss.ptr(snap[j]),
                                              ss.ptr(grads[0]), losses.data_ptr() + 4 * li, ctypes.c_void_p(st)))
                mb, li = mb + 1, li + 1
                g.asp_push(j, grads[0], base[j])
        e1.record(stream)
        g.sync()
        ms = e0.elapsed_time(e1)
        st_ = g.stats(64)
        w_end = g.params()
        g.close()
        return ms, st_, w_end

    for _ in range(max(args.warmup, 1)):
        one_run()
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    runs = [one_run() for _ in range(args.steps)]
    clk = clocks.stop()
    ms = sum(r[0] for r in runs)
    updates = (bsp_steps + asp_pushes) * args.steps
    lv = losses.cpu().numpy()
    st, w_end = runs[-1][1], runs[-1][2]
    # held-out evaluation of the final parameters (reporting only; not part of the timed path)
    Wm = w_end.reshape(d, C).astype(np.float64)
    test_acc = float(np.mean(np.argmax(Xte @ Wm, 1) == yte))
    train_acc = float(np.mean(np.argmax(X @ Wm, 1) == y))
    k_sw = n * bsp_steps                       # losses of the BSP phase come first (n per superstep)
    line = {"metric": METRIC, "value": round(updates / (ms / 1e3), 1),
            "unit": "protocol updates/s (BSP supersteps + ASP pushes, each with its softmax_grad kernel(s))",
            "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 1), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian-mixture toy dataset, inputs/toy_dataset)",
            "config": {"workload": cfg["name"], "P": P, "n_workers": n, "n_shards": S, "batch": B,
                       "bsp_steps": bsp_steps, "asp_pushes": asp_pushes, "asp_window_events": 1,
                       "note": "a step = one whole training run from w = 0"},
            "training": {"loss_first": float(lv[0]), "loss_first10_mean": float(lv[:10].mean()),
                         "loss_at_switch_last10_bsp_mean": float(lv[k_sw - 10:k_sw].mean()),
                         "loss_last10_mean": float(lv[-10:].mean()),
                         "test_accuracy": test_acc, "train_accuracy": train_acc,
                         "data_recipe": {k: (round(v, 6) if isinstance(v, float) else v) for k, v in TOY_RECIPE.items()},
                         "loss_every_10th_update": [round(float(x), 5) for x in lv[::10]],
                         "version": st["version"], "staleness_hist": {str(i): int(x) for i, x in enumerate(st["hist"])
                                                                      if x}},
            "clocks": clk}
    emit(line)


# ------------------------------------------------------------------------------------------------------------------
# --workload: sync-only time of the whole 64K-iteration training workload (the sync-path
# analog of Table II's throughput column): pure BSP, pure ASP and switched at s, each with the Table I
# workload-preserving remap of steps and lr-decay boundaries (DESIGN reading C11).
WORKLOADS = {
    # W samples, B per worker, switch point s = num/den of W (P:1552 for config 3's 12.5%), decay boundaries W_i in
    # samples with their factors (config 2: ResNet-32 on CIFAR-10's decays at 50% and 75% of W; config 3 uses the same
    # step-decay shape, reading C27)
    "2": dict(W=64000 * 128, B=128, s=(1, 16), Wb=[32000 * 128, 48000 * 128], factors=[0.1, 0.01]),
    "3": dict(W=64000 * 128, B=128, s=(1, 8), Wb=[32000 * 128, 48000 * 128], factors=[0.1, 0.01]),
}


def asp_workload_events(n: int, n_push: int, ver0: int, jitter: int = 100, seed: int = 7, period: int = 1000):
    """Arrival order of an ASP phase from the seeded integer-tick schedule (ss_schedule, DESIGN reading C7: every
    worker pulls at t = 0, then each push is followed by the pusher's pull) with the version each worker sends: the
    version of its last pull. Returns (kind, worker, version) int arrays; the phase starts at ver0."""
    import numpy as np
    from paper_2104_08364_b200 import syncswitch as ss
    s, (kind, worker, _) = ss.ss_schedule(n, [period] * n, n_push, jitter=jitter, seed=seed)
    ss.ss_check(s)
    version = np.zeros(kind.size, dtype=np.int64)
    base = [ver0] * n
    ver = ver0
    for e in range(kind.size):
        j = int(worker[e])
        if kind[e] == 1:
            base[j] = ver
            version[e] = ver
        else:
            version[e] = base[j]
            ver += 1
    return kind, worker, version


def run_workload(args):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2104_08364_b200 import syncswitch as ss

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, wl = CONFIGS[args.config], WORKLOADS[args.config]
    P, n, S, win = cfg["P"], cfg["n"], cfg["S"], args.window or cfg["window"]
    hosted = [j for j in range(n) if (j * world) // n == rank]
    # exchange: one worker per GPU or fewer (the paper's layout) -> the one-kernel pull exchange (mode 3); more workers
    # than GPUs -> each rank pre-sums its workers and scatters one slice per owner (mode 2)
    fused = (3 if n <= world else 2) if args.fused == "auto" else int(args.fused)
    w0 = torch.empty(P, device="cuda")
    ss.ss_check(ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0))
    w0.mul_(64.0)
    ring = {(j, r): torch.empty(P, device="cuda") for j in hosted for r in range(2)}
    for (j, r), buf in ring.items():
        ss.ss_check(ss.ss_synth_grad(SEED, j, r, 0, P, buf))
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def one_run(s_num, s_den, scale=1):
        """One whole workload (steps / scale) from a fresh context; returns the run's record."""
        s, (n_bsp, n_asp, bounds) = ss.ss_table1(wl["W"], wl["B"], n, s_num, s_den, wl["Wb"])
        ss.ss_check(s)
        n_bsp, n_asp = n_bsp // scale, n_asp // scale
        g = ss.SyncSwitch(w0, S, n, 0.1, 0.9)
        if world > 1:
            uid = [ss.ss_nccl_unique_id() if rank == 0 else None]      # one NCCL id per communicator
            dist.broadcast_object_list(uid, src=0)
            g.init_dist(rank, world, uid[0])
            g.set_fused(fused)
        g.set_window(win)
        g.set_lr_schedule(bounds, wl["factors"])
        if world > 1 and fused:
            dst = {j: g.pull_buffer(j) for j in hosted}
        else:
            dst = {j: ss.ptr(t) for j, t in pull_bufs.items()}
        # BSP supersteps: step t feeds ring slot t mod 2 of every hosted worker
        gp = [(ctypes.c_void_p * max(len(hosted), 1))(*[ss.ptr(ring[(j, r)]) for j in hosted]) for r in range(2)]
        ws = np.array(hosted, dtype=np.int32)
        vs = np.zeros(max(len(hosted), 1), dtype=np.int64)
        kind, worker, version = asp_workload_events(n, n_asp, n_bsp)
        evs = (ss.ss_event * max(kind.size, 1))()
        cnt = [0] * n
        for e in range(kind.size):
            j = int(worker[e])
            if kind[e] == 0:
                buf = ring.get((j, cnt[j] % 2))
                cnt[j] += 1
                evs[e] = ss.ss_event(0, j, int(version[e]), ss.ptr(buf) if buf is not None else None, None)
            else:
                evs[e] = ss.ss_event(1, j, int(version[e]), None, dst.get(j))
        stream = torch.cuda.ExternalStream(g.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        L, c = ss.lib, g.ctx
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for t in range(n_bsp):
            vs[:] = t
            st = L.ss_bsp_step(c, ctypes.cast(gp[t % 2], ctypes.c_void_p), ws.ctypes.data, vs.ctypes.data,
                               len(hosted))
            st = st or L.ss_flush(c)         # the next superstep's gradients depend on this one
            if st:
                raise ss.SSError(st, g.last_error())
        if n_asp:
            ss.ss_check(L.ss_switch(c, ss.SS_ASP, 0))
            st = L.ss_asp_replay(c, ctypes.cast(evs, ctypes.c_void_p), kind.size, None)
            if st:
                raise ss.SSError(st, g.last_error())
        g.sync()
        e1.record(stream)
        barrier()
        wall = time.perf_counter() - t0
        tt = torch.tensor([e0.elapsed_time(e1) / 1e3, wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_s, wall_s = tt.tolist()
        stt = g.stats(256)
        assert stt["status"] == 0 and stt["version"] == n_bsp + n_asp, (stt, g.last_error())
        hist = [int(x) for x in stt["hist"]]
        top = max((i for i, x in enumerate(hist) if x), default=0)
        g.close()
        return {"s": f"{s_num}/{s_den}", "bsp_steps": n_bsp, "asp_pushes": n_asp, "lr_boundaries_version": bounds,
                "seconds": dev_s, "wall_seconds": wall_s, "samples_per_s": wl["W"] / scale / dev_s,
                "staleness_hist": {str(i): hist[i] for i in range(top + 1) if hist[i]},
                "max_staleness": top}

    pull_bufs = {} if (world > 1 and fused) else {j: torch.empty(P, device="cuda") for j in hosted}
    one_run(1, 2, scale=100)                         # warm-up: kernels loaded, peer mappings exercised
    clocks = Clocks(local)
    clocks.start()
    runs = {"bsp": one_run(1, 1), "asp": one_run(0, 1), "switched": one_run(*wl["s"])}
    clk = clocks.stop()
    sw = runs["switched"]
    line = {"metric": METRIC, "value": round(sw["seconds"], 4),
            "unit": "s of sync-only time for the whole workload (switched protocol)", "n_gpus": world,
            "steps": sw["bsp_steps"] + sw["asp_pushes"], "warmup": 1, "ms_per_step": None,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded counter-hash gradients, 2-slot rings per worker)",
            "config": {"workload": cfg["name"] + f"; whole workload W={wl['W']} samples, B={wl['B']}, switched at "
                                                 f"s={wl['s'][0]}/{wl['s'][1]} (Table I remap)",
                       "P": P, "n_workers": n, "n_shards": S, "asp_window_events": win,
                       "exchange": "single GPU" if world == 1 else
                       ["NCCL RS/AG + send/recv", "fused peer-memory, exact", "fused peer-memory, pre-summed",
                    "fused one-kernel pull (gradient buffers read in place over NVLink)"][fused],
                       "schedule": "ss_schedule, period 1000 ticks, jitter 100, seed 7; each push followed by its pull"},
            "runs": runs,
            "speedup_vs_bsp": {k: runs["bsp"]["seconds"] / r["seconds"] for k, r in runs.items()},
            "clocks": clk}
    if rank == 0:
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _oracle_step(orc, o, n, grads_bsp, grads_asp):
    ver = o.version
    assert o.bsp_step(grads_bsp, versions=[ver] * n) == 0
    o.switch(orc.ASP, 0)
    for j in range(n):
        rc, st = o.asp_push(j, grads_asp[j], ver + 1)
        assert rc == 0 and st == j
        o.pull(j)
    o.switch(orc.BSP, 0)


def _oracle_inputs(orc, n, P):
    import numpy as np
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    gb = [orc.synth_grad(SEED, j, 0, 0, P) for j in range(n)]
    ga = [orc.synth_grad(SEED, j, 1, 0, P) for j in range(n)]
    return w0, gb, ga


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, seconds: float):
    """The oracle as it stands (single-threaded C), on this host, on a bounded sample: full-size steps until
    `seconds` of CPU work (at least one)."""
    import oracle as orc
    orc.build()
    P, n, S = cfg["P"], cfg["n"], cfg["S"]
    w0, gb, ga = _oracle_inputs(orc, n, P)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    t0 = time.perf_counter()
    k = 0
    while True:
        _oracle_step(orc, o, n, gb, ga)
        k += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": k / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{k} full-size steps of the same workload ({el:.1f} s, P={P}, n={n})",
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}


def run_reference(args):
    """--impl reference: the oracle as it stands on the host's cores, on the same config / metric / unit. Each step is
    the same step on a bounded sample: the first P_s elements of the parameter vector (the path is elementwise, cost
    linear in P), with P_s sized so the K + W steps take ~2 minutes; value = full-workload steps/s."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and rank != 0:
        return
    import oracle as orc
    orc.build()
    cfg = CONFIGS[args.config]
    P, n, S = cfg["P"], cfg["n"], cfg["S"]
    # calibrate on a 1M-element slice
    Pc = min(P, 1 << 20)
    w0, gb, ga = _oracle_inputs(orc, n, Pc)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    t0 = time.perf_counter()
    _oracle_step(orc, o, n, gb, ga)
    per_elem = (time.perf_counter() - t0) / Pc
    budget = 120.0 / max(args.steps + args.warmup, 1)
    Ps = int(max(4096, min(P, budget / per_elem)))
    w0, gb, ga = _oracle_inputs(orc, n, Ps)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    for _ in range(args.warmup):
        _oracle_step(orc, o, n, gb, ga)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _oracle_step(orc, o, n, gb, ga)
    el = time.perf_counter() - t0
    value = args.steps / el * (Ps / P)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded counter-hash gradients)",
            "impl": "reference",
            "config": {"workload": cfg["name"], "P": P, "n_workers": n, "n_shards": S},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
                             "host_cpus": os.cpu_count(),
                             "sample": f"each step on the first {Ps} of {P} elements ({Ps / P:.4f} of the vector), "
                                       f"scaled by P/P_s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _self_launch(a) -> int:
    """`--gpus N > 1` from a plain shell (no WORLD_SIZE in the environment): start the N ranks with
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1) running this same command line. Rank 0
    prints the JSON line on the shared stdout; torchrun's own messages go to stderr."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = {**os.environ, "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS", "1")}
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        sys.exit(_self_launch(a))
    _claim_stdout()
    if a.impl == "reference":
        run_reference(a)
    elif a.config == "4":
        run_scenario(a)
    elif a.config == "1":
        run_toy(a)
    elif a.workload:
        run_workload(a)
    else:
        run_ours(a)
