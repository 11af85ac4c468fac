"""Thin ctypes binding of the C-ABI in include/syncswitch.h (libsyncswitch.so, built in-tree for sm_100a).

Argument marshalling only: every step of the synchronization path runs in the library's CUDA kernels and NCCL calls.
There is no Python or CPU fallback — importing this module fails loudly when the shared library is missing, and
calls that need a GPU fail with SS_E_CUDA when there is none.

Functions keep the C names (``ss_init``, ``ss_bsp_step``, ``ss_asp_push``, ``ss_pull``, ``ss_switch``, …). Buffers
may be torch tensors (CUDA or CPU; CPU tensors are host memory, staged by the library), numpy arrays (host memory)
or raw integer addresses. ``SyncSwitch`` wraps a context with the same method names minus the ``ss_`` prefix.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SS_LIB_VARIANT") or os.path.join(_PKG, "libsyncswitch.so")   # variant: tuning sweeps

SS_BSP, SS_ASP = 0, 1
STATUS = ["SS_OK", "SS_E_INVAL", "SS_E_STATE", "SS_E_PROTOCOL", "SS_E_BARRIER", "SS_E_CAUSALITY", "SS_E_DIVERGED",
          "SS_E_CUDA", "SS_E_NCCL", "SS_E_OOM"]
(SS_OK, SS_E_INVAL, SS_E_STATE, SS_E_PROTOCOL, SS_E_BARRIER, SS_E_CAUSALITY, SS_E_DIVERGED, SS_E_CUDA, SS_E_NCCL,
 SS_E_OOM) = range(10)

# every symbol include/syncswitch.h declares (tests check the library exports each one)
EXPORTS = ["ss_init", "ss_init_dist", "ss_nccl_unique_id", "ss_destroy", "ss_last_error", "ss_set_lr_schedule",
           "ss_set_lr_policy", "ss_current_lr", "ss_bsp_step", "ss_asp_push", "ss_pull", "ss_switch",
           "ss_asp_replay", "ss_sync", "ss_flush", "ss_read_params", "ss_read_velocity", "ss_get_stats", "ss_get_log",
           "ss_set_window", "ss_get_stream", "ss_wait_stream", "ss_profile", "ss_kernel_stats", "ss_synth_grad",
           "ss_softmax_grad", "ss_table1", "ss_schedule", "ss_detector_new", "ss_detector_window",
           "ss_detector_free", "ss_greedy_decision", "ss_route_plan", "ss_set_fused", "ss_set_nesterov", "ss_get_exchange", "ss_pull_buffer", "ss_grad_buffer",
           "ss_scenario_run", "ss_set_momentum_policy", "ss_set_members", "ss_detector_window_masked",
           "ss_dynamic_criterion", "ss_criterion_observe", "ss_capture_begin", "ss_capture_end",
           "ss_capture_replay"]


class SSError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")


class ss_route_op(ctypes.Structure):
    _fields_ = [("window", ctypes.c_int32), ("phase", ctypes.c_int32), ("op", ctypes.c_int32),
                ("peer", ctypes.c_int32), ("event", ctypes.c_int32), ("offset", ctypes.c_int64),
                ("count", ctypes.c_int64)]


class ss_scenario(ctypes.Structure):
    _fields_ = [("n_workers", ctypes.c_int32), ("batch", ctypes.c_int64), ("total_samples", ctypes.c_int64),
                ("quota_num", ctypes.c_int64), ("quota_den", ctypes.c_int64), ("period", ctypes.c_int64),
                ("jitter", ctypes.c_int64), ("sched_seed", ctypes.c_uint64), ("grad_seed", ctypes.c_uint64),
                ("slow_worker", ctypes.c_int32), ("slow_factor", ctypes.c_int64), ("slow_t0", ctypes.c_int64),
                ("slow_t1", ctypes.c_int64), ("window_ticks", ctypes.c_int64), ("K", ctypes.c_int32),
                ("policy", ctypes.c_int32)]


class ss_switch_event(ctypes.Structure):
    _fields_ = [("tick", ctypes.c_int64), ("version", ctypes.c_int64), ("to_protocol", ctypes.c_int32),
                ("reason", ctypes.c_int32), ("members", ctypes.c_int32)]


class ss_scenario_result(ctypes.Structure):
    _fields_ = [("bsp_steps", ctypes.c_int64), ("asp_pushes", ctypes.c_int64), ("dropped", ctypes.c_int64),
                ("end_tick", ctypes.c_int64), ("version", ctypes.c_int64), ("windows", ctypes.c_int64),
                ("n_switches", ctypes.c_int32)]


class ss_event(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("worker", ctypes.c_int32), ("version", ctypes.c_int64),
                ("grad", ctypes.c_void_p), ("dst", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2104_08364_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i32, i64, u64, f32, f64, p = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double,
                                  ctypes.c_void_p)
    sig = {
        "ss_init": [p, p, i64, i32, i32, f32, f32],
        "ss_init_dist": [p, i32, i32, p],
        "ss_set_fused": [p, i32],
        "ss_get_exchange": [p, p, p],
        "ss_set_nesterov": [p, i32],
        "ss_pull_buffer": [p, i32, p],
        "ss_grad_buffer": [p, i32, p],
        "ss_nccl_unique_id": [p],
        "ss_set_lr_schedule": [p, p, p, i32],
        "ss_set_lr_policy": [p, i32, f32],
        "ss_set_momentum_policy": [p, i32, i64, i64],
        "ss_set_members": [p, p, i32],
        "ss_detector_window_masked": [p, p, p, p, p, p],
        "ss_current_lr": [p, i32, p],
        "ss_bsp_step": [p, p, p, p, i32],
        "ss_asp_push": [p, i32, p, i64, p],
        "ss_pull": [p, i32, p, p],
        "ss_switch": [p, i32, i64],
        "ss_asp_replay": [p, p, i64, p],
        "ss_sync": [p],
        "ss_flush": [p],
        "ss_read_params": [p, p],
        "ss_read_velocity": [p, p],
        "ss_get_stats": [p, p, p, p, i32, p],
        "ss_get_log": [p, p, i64, p],
        "ss_set_window": [p, i32],
        "ss_capture_begin": [p],
        "ss_capture_end": [p, p],
        "ss_capture_replay": [p, i64],
        "ss_get_stream": [p, p],
        "ss_wait_stream": [p, p],
        "ss_profile": [p, i32],
        "ss_kernel_stats": [p, i32, p, p, p, p],
        "ss_synth_grad": [u64, i32, i64, i64, i64, p, p],
        "ss_softmax_grad": [p, p, i32, i32, i32, p, p, p, p],
        "ss_dynamic_criterion": [p, p, i32, i32, i32, p, p, p, p, p],
        "ss_table1": [i64, i64, i64, i64, i64, p, i32, p, p, p],
        "ss_schedule": [i32, p, i64, u64, i32, i64, i64, i64, i64, p, p, p, p],
        "ss_detector_new": [p, i32, i32],
        "ss_detector_window": [p, p, p, p, p],
        "ss_route_plan": [i32, i32, i32, i32, i64, i32, i32, p, p, i64, p, i64, p, p],
        "ss_scenario_run": [p, p, p, p, i32],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.ss_destroy.argtypes = [p]
    L.ss_destroy.restype = None
    L.ss_detector_free.argtypes = [p]
    L.ss_detector_free.restype = None
    L.ss_last_error.argtypes = [p]
    L.ss_last_error.restype = ctypes.c_char_p
    L.ss_criterion_observe.argtypes = [p, f32, f32, f32, i32]
    L.ss_criterion_observe.restype = i32
    L.ss_greedy_decision.argtypes = [i32, i32, i32, i64, i64]
    L.ss_greedy_decision.restype = i32
    return L


lib = _load()


def ptr(x) -> int | None:
    """Address of a torch tensor / numpy array / int (None -> NULL). No copies: buffers must be contiguous."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "numpy buffers must be C-contiguous"
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensors must be contiguous"
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


def _a(arr, dtype):
    return np.ascontiguousarray(arr, dtype=dtype)


# ------------------------------------------------------------------------------------------------------------------
# C names
def ss_init(params, n_params: int, n_shards: int, n_workers: int, lr: float, momentum: float):
    h = ctypes.c_void_p()
    s = lib.ss_init(ctypes.byref(h), ptr(params), n_params, n_shards, n_workers, lr, momentum)
    return s, h.value


def ss_last_error(ctx) -> str:
    return lib.ss_last_error(ctx).decode()


def ss_check(status: int, ctx=None):
    if status != SS_OK:
        raise SSError(status, ss_last_error(ctx) if ctx else "")
    return status


def ss_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    ss_check(lib.ss_nccl_unique_id(buf))
    return buf.raw


def ss_init_dist(ctx, rank: int, world: int, uid: bytes) -> int:
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    return lib.ss_init_dist(ctx, rank, world, buf)


def ss_bsp_step(ctx, grads, workers, versions) -> int:
    k = len(grads)
    gp = (ctypes.c_void_p * max(k, 1))(*[ptr(g) for g in grads])
    w = _a(workers, np.int32)
    v = _a(versions, np.int64)
    return lib.ss_bsp_step(ctx, ctypes.cast(gp, ctypes.c_void_p), w.ctypes.data, v.ctypes.data, k)


def ss_asp_push(ctx, worker: int, grad, version: int):
    st = ctypes.c_int64(-1)
    s = lib.ss_asp_push(ctx, worker, ptr(grad), version, ctypes.byref(st))
    return s, st.value


def ss_pull(ctx, worker: int, dst):
    ver = ctypes.c_int64(-1)
    s = lib.ss_pull(ctx, worker, ptr(dst), ctypes.byref(ver))
    return s, ver.value


def ss_switch(ctx, protocol: int, at_step: int) -> int:
    return lib.ss_switch(ctx, protocol, at_step)


def ss_asp_replay(ctx, events):
    """events: iterable of (kind, worker, version, grad, dst)."""
    events = list(events)
    arr = (ss_event * max(len(events), 1))()
    for i, (kind, worker, version, grad, dst) in enumerate(events):
        arr[i] = ss_event(kind, worker, version, ptr(grad), ptr(dst))
    out = np.zeros(max(len(events), 1), dtype=np.int64)
    s = lib.ss_asp_replay(ctx, ctypes.cast(arr, ctypes.c_void_p), len(events), out.ctypes.data)
    return s, out[:len(events)]


def ss_sync(ctx) -> int:
    return lib.ss_sync(ctx)


def ss_flush(ctx) -> int:
    return lib.ss_flush(ctx)


def ss_read_params(ctx, n_params: int):
    out = np.empty(n_params, dtype=np.float32)
    s = lib.ss_read_params(ctx, out.ctypes.data)
    return s, out


def ss_read_velocity(ctx, n_params: int):
    out = np.empty(n_params, dtype=np.float32)
    s = lib.ss_read_velocity(ctx, out.ctypes.data)
    return s, out


def ss_get_stats(ctx, hist_len: int = 64):
    ver, proto, dropped = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_uint64()
    hist = np.zeros(hist_len, dtype=np.uint64)
    s = lib.ss_get_stats(ctx, ctypes.byref(ver), ctypes.byref(proto), hist.ctypes.data, hist_len,
                         ctypes.byref(dropped))
    return s, dict(version=ver.value, protocol=proto.value, hist=hist, dropped=dropped.value)


def ss_get_log(ctx):
    total = ctypes.c_int64()
    lib.ss_get_log(ctx, None, 0, ctypes.byref(total))
    out = np.zeros((total.value, 4), dtype=np.int64)
    s = lib.ss_get_log(ctx, out.ctypes.data if total.value else None, total.value, ctypes.byref(total))
    return s, out


def ss_set_lr_schedule(ctx, boundaries, factors) -> int:
    b = _a(boundaries, np.int64)
    f = _a(factors, np.float32)
    return lib.ss_set_lr_schedule(ctx, b.ctypes.data if b.size else None, f.ctypes.data if f.size else None, b.size)


def ss_set_lr_policy(ctx, asp_rule: int, weight_decay: float) -> int:
    return lib.ss_set_lr_policy(ctx, asp_rule, weight_decay)


def ss_current_lr(ctx, protocol: int) -> float:
    out = ctypes.c_float()
    ss_check(lib.ss_current_lr(ctx, protocol, ctypes.byref(out)), ctx)
    return out.value


def ss_set_window(ctx, max_events: int) -> int:
    return lib.ss_set_window(ctx, max_events)


def ss_get_stream(ctx) -> int:
    s = ctypes.c_void_p()
    ss_check(lib.ss_get_stream(ctx, ctypes.byref(s)), ctx)
    return s.value or 0


def ss_wait_stream(ctx, stream: int) -> int:
    return lib.ss_wait_stream(ctx, stream)


def ss_profile(ctx, on: bool) -> int:
    return lib.ss_profile(ctx, int(on))


def ss_kernel_stats(ctx, kernel_id: int):
    n, ms, by, nv = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    ss_check(lib.ss_kernel_stats(ctx, kernel_id, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by),
                                 ctypes.byref(nv)), ctx)
    return dict(launches=n.value, ms=ms.value, bytes=by.value, nvlink_bytes=nv.value)


def ss_destroy(ctx) -> None:
    lib.ss_destroy(ctx)


def ss_synth_grad(seed: int, j: int, k: int, i0: int, count: int, dst, stream: int = 0) -> int:
    return lib.ss_synth_grad(seed, j, k, i0, count, ptr(dst), stream or None)


def ss_softmax_grad(X, y, B: int, d: int, C: int, W, grad, loss, stream: int = 0) -> int:
    return lib.ss_softmax_grad(ptr(X), ptr(y), B, d, C, ptr(W), ptr(grad), ptr(loss), stream or None)


def ss_dynamic_criterion(X, y, B: int, d: int, C: int, W, g_prev, g_out, stats, stream: int = 0) -> int:
    return lib.ss_dynamic_criterion(ptr(X), ptr(y), B, d, C, ptr(W), ptr(g_prev), ptr(g_out), ptr(stats),
                                    stream or None)


class CriterionRule:
    """ss_criterion_observe: fires after T consecutive steps with |Delta| < c sigma."""

    def __init__(self, c: float = 2.0, T: int = 5):
        self.c, self.T, self._run = c, T, ctypes.c_int32(0)

    def observe(self, norm_delta: float, sigma: float) -> bool:
        return bool(lib.ss_criterion_observe(ctypes.byref(self._run), norm_delta, sigma, self.c, self.T))


def ss_table1(W: int, B: int, N: int, s_num: int, s_den: int, Wb):
    Wb = _a(Wb, np.int64)
    out = np.zeros(max(Wb.size, 1), dtype=np.int64)
    bsp, asp = ctypes.c_int64(), ctypes.c_int64()
    s = lib.ss_table1(W, B, N, s_num, s_den, Wb.ctypes.data if Wb.size else None, Wb.size, ctypes.byref(bsp),
                      ctypes.byref(asp), out.ctypes.data)
    return s, (bsp.value, asp.value, [int(x) for x in out[:Wb.size]])


def ss_schedule(n: int, period, n_push: int, jitter: int = 0, seed: int = 7, slow_worker: int = -1,
                slow_factor: int = 1, slow_t0: int = 0, slow_t1: int = 0):
    per = _a(period, np.int64)
    cap = n + 2 * n_push
    kind = np.zeros(cap, dtype=np.int32)
    worker = np.zeros(cap, dtype=np.int32)
    tick = np.zeros(cap, dtype=np.int64)
    ne = ctypes.c_int64()
    s = lib.ss_schedule(n, per.ctypes.data, jitter, seed, slow_worker, slow_factor, slow_t0, slow_t1, n_push,
                        kind.ctypes.data, worker.ctypes.data, tick.ctypes.data, ctypes.byref(ne))
    return s, (kind[:ne.value], worker[:ne.value], tick[:ne.value])


def ss_route_plan(rank: int, world: int, n_workers: int, n_shards: int, n_params: int, max_window: int, fused: bool,
                  kind, worker):
    """Routing plan of an ASP event sequence as `rank` executes it: (status, [(window, phase, op, peer, event,
    offset, count)], n_windows)."""
    k = _a(kind, np.int32)
    w = _a(worker, np.int32)
    total, nwin = ctypes.c_int64(), ctypes.c_int32()
    s = lib.ss_route_plan(rank, world, n_workers, n_shards, n_params, max_window, int(fused), k.ctypes.data,
                          w.ctypes.data, k.size, None, 0, ctypes.byref(total), ctypes.byref(nwin))
    if s != SS_OK:
        return s, [], 0
    arr = (ss_route_op * max(total.value, 1))()
    s = lib.ss_route_plan(rank, world, n_workers, n_shards, n_params, max_window, int(fused), k.ctypes.data,
                          w.ctypes.data, k.size, ctypes.cast(arr, ctypes.c_void_p), total.value, ctypes.byref(total),
                          ctypes.byref(nwin))
    ops = [(o.window, o.phase, o.op, o.peer, o.event, o.offset, o.count) for o in arr[:total.value]]
    return s, ops, nwin.value


def ss_scenario_run(ctx, sc: dict, cap: int = 256):
    """Config-4 scenario on a context (or ctx=None: host-only dry run). Returns (status, switch log
    [(tick, version, to, reason)], result dict)."""
    c = ss_scenario(**sc)
    log = (ss_switch_event * cap)()
    out = ss_scenario_result()
    s = lib.ss_scenario_run(ctx, ctypes.byref(c), ctypes.byref(out), ctypes.cast(log, ctypes.c_void_p), cap)
    res = {k: getattr(out, k) for k, _ in ss_scenario_result._fields_}
    entries = [(e.tick, e.version, e.to_protocol, e.reason, e.members) for e in log[:min(out.n_switches, cap)]]
    return s, entries, res


class Detector:
    """ss_detector_* (P:1425)."""

    def __init__(self, n: int, K: int = 3):
        h = ctypes.c_void_p()
        ss_check(lib.ss_detector_new(ctypes.byref(h), n, K))
        self._h, self.n = h.value, n

    def window(self, samples, busy, mask=None):
        s = _a(samples, np.float64)
        b = _a(busy, np.float64)
        m = _a(mask, np.uint8) if mask is not None else None
        flag = np.zeros(self.n, dtype=np.int32)
        clean = ctypes.c_int32()
        ss_check(lib.ss_detector_window_masked(self._h, s.ctypes.data, b.ctypes.data,
                                               m.ctypes.data if m is not None else None, flag.ctypes.data,
                                               ctypes.byref(clean)))
        return flag.astype(bool), bool(clean.value)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ss_detector_free(self._h)
            self._h = None


def ss_greedy_decision(protocol: int, any_straggler: bool, cluster_clean: bool, bsp_done: int, bsp_quota: int) -> int:
    return int(lib.ss_greedy_decision(protocol, int(any_straggler), int(cluster_clean), bsp_done, bsp_quota))


# ------------------------------------------------------------------------------------------------------------------
class SyncSwitch:
    """One context: ``SyncSwitch(params, n_shards, n_workers, lr, momentum)``; methods raise SSError on failure
    (``*_status`` variants of the protocol calls return the raw status instead)."""

    def __init__(self, params, n_shards: int, n_workers: int, lr: float, momentum: float, n_params: int | None = None):
        if n_params is None:
            n_params = int(params.numel() if hasattr(params, "numel") else np.asarray(params).size)
        self.P, self.n, self.S = n_params, n_workers, n_shards
        self._destroy = lib.ss_destroy   # held by the instance: still callable during interpreter shutdown
        s, self.ctx = ss_init(params, n_params, n_shards, n_workers, lr, momentum)
        if s != SS_OK:
            raise SSError(s, "ss_init failed")

    def close(self):
        if getattr(self, "ctx", None):
            self._destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _chk(self, s):
        return ss_check(s, self.ctx)

    def init_dist(self, rank: int, world: int, uid: bytes):
        return self._chk(ss_init_dist(self.ctx, rank, world, uid))

    def set_fused(self, mode: int):
        return self._chk(lib.ss_set_fused(self.ctx, mode))

    def exchange(self) -> dict:
        m, v = ctypes.c_int32(), ctypes.c_int32()
        self._chk(lib.ss_get_exchange(self.ctx, ctypes.byref(m), ctypes.byref(v)))
        return {"fused": m.value, "nvls": bool(v.value)}

    def pull_buffer(self, worker: int) -> int:
        out = ctypes.c_void_p()
        self._chk(lib.ss_pull_buffer(self.ctx, worker, ctypes.byref(out)))
        return out.value

    def grad_buffer(self, worker: int) -> int:
        """Address of the exported gradient buffer of a hosted worker (fused mode 3 reads it in place)."""
        out = ctypes.c_void_p()
        self._chk(lib.ss_grad_buffer(self.ctx, worker, ctypes.byref(out)))
        return out.value

    def set_lr_schedule(self, boundaries, factors):
        return self._chk(ss_set_lr_schedule(self.ctx, boundaries, factors))

    def set_lr_policy(self, asp_rule: int, weight_decay: float = 0.0):
        return self._chk(ss_set_lr_policy(self.ctx, asp_rule, weight_decay))

    def set_members(self, workers):
        w = _a(workers, np.int32)
        return self._chk(lib.ss_set_members(self.ctx, w.ctypes.data, w.size))

    def set_nesterov(self, on: bool):
        return self._chk(lib.ss_set_nesterov(self.ctx, int(on)))

    def set_momentum_policy(self, rule: int, samples_per_epoch: int = 1, batch: int = 1):
        return self._chk(lib.ss_set_momentum_policy(self.ctx, rule, samples_per_epoch, batch))

    def current_lr(self, protocol: int) -> float:
        return ss_current_lr(self.ctx, protocol)

    def bsp_step_status(self, grads, workers=None, versions=None) -> int:
        if workers is None:
            workers = list(range(len(grads)))
        if versions is None:
            versions = [self.version] * len(grads)
        return ss_bsp_step(self.ctx, grads, workers, versions)

    def bsp_step(self, grads, workers=None, versions=None):
        return self._chk(self.bsp_step_status(grads, workers, versions))

    def asp_push_status(self, worker: int, grad, version: int):
        return ss_asp_push(self.ctx, worker, grad, version)

    def asp_push(self, worker: int, grad, version: int) -> int:
        s, st = ss_asp_push(self.ctx, worker, grad, version)
        self._chk(s)
        return st

    def pull(self, worker: int, dst=None) -> int:
        s, ver = ss_pull(self.ctx, worker, dst)
        self._chk(s)
        return ver

    def switch(self, protocol: int, at_step: int):
        return self._chk(ss_switch(self.ctx, protocol, at_step))

    def switch_status(self, protocol: int, at_step: int) -> int:
        return ss_switch(self.ctx, protocol, at_step)

    def asp_replay(self, events):
        s, out = ss_asp_replay(self.ctx, events)
        self._chk(s)
        return out

    def sync(self):
        return self._chk(ss_sync(self.ctx))

    def flush(self):
        return self._chk(ss_flush(self.ctx))

    def sync_status(self) -> int:
        return ss_sync(self.ctx)

    def params(self) -> np.ndarray:
        s, out = ss_read_params(self.ctx, self.P)
        if s not in (SS_OK, SS_E_DIVERGED):
            self._chk(s)
        return out

    def velocity(self) -> np.ndarray:
        s, out = ss_read_velocity(self.ctx, self.P)
        if s not in (SS_OK, SS_E_DIVERGED):
            self._chk(s)
        return out

    def stats(self, hist_len: int = 64) -> dict:
        s, d = ss_get_stats(self.ctx, hist_len)
        d["status"] = s
        return d

    @property
    def version(self) -> int:
        return self.stats(1)["version"]

    def log(self) -> np.ndarray:
        return ss_get_log(self.ctx)[1]

    def capture_begin(self):
        return self._chk(lib.ss_capture_begin(self.ctx))

    def capture_end(self) -> int:
        dv = ctypes.c_int64()
        self._chk(lib.ss_capture_end(self.ctx, ctypes.byref(dv)))
        return dv.value

    def capture_replay(self, times: int):
        return self._chk(lib.ss_capture_replay(self.ctx, times))

    def set_window(self, k: int):
        return self._chk(ss_set_window(self.ctx, k))

    @property
    def stream(self) -> int:
        return ss_get_stream(self.ctx)

    def wait_stream(self, stream: int):
        return self._chk(ss_wait_stream(self.ctx, stream))

    def profile(self, on: bool):
        return self._chk(ss_profile(self.ctx, on))

    def kernel_stats(self, kernel_id: int) -> dict:
        return ss_kernel_stats(self.ctx, kernel_id)

    def last_error(self) -> str:
        return ss_last_error(self.ctx)
