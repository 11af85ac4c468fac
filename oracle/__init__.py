"""CPU oracle for the Sync-Switch synchronization path (ctypes binding over oracle/oracle.c).

TEST INFRASTRUCTURE ONLY. Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path (``paper_2104_08364_b200``) never does, and
this package never imports the product path: the two share no code.

Every wrapped function follows a cited passage of PAPER.md; see oracle/oracle.h and DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle_state.inc", "oracle.h")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, E_INVAL, E_STATE, E_PROTOCOL, E_BARRIER, E_CAUSALITY, E_DIVERGED = range(7)
BSP, ASP = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no contraction, no fast-math: float arithmetic is exactly as written)."""
    stale = not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB_PATH) for s in _SRC)
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
            "-Wall", "-Wextra", "-Wno-unused-parameter",
            os.path.join(_HERE, "oracle.c"), "-lm", "-o", tmp])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None

_i32, _i64, _u64, _f32, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double
_p = ctypes.c_void_p


def lib():
    global _lib
    if _lib is not None:
        return _lib
    L = ctypes.CDLL(build())
    L.orc_shard_pad.restype = _i64
    L.orc_shard_pad.argtypes = [_i64, _i32]
    L.orc_shard_offsets.argtypes = [_i64, _i32, _p]
    L.orc_shard_owner.restype = _i32
    L.orc_shard_owner.argtypes = [_i32, _i32, _i32]
    L.orc_worker_host.restype = _i32
    L.orc_worker_host.argtypes = [_i32, _i32, _i32]
    L.orc_lr_factor.restype = _f64
    L.orc_lr_factor.argtypes = [_i64, _p, _p, _i32]
    L.orc_lr.restype = _f32
    L.orc_lr.argtypes = [_f32, _f64, _i32, _i32, _i32]
    L.orc_table1.restype = _i32
    L.orc_table1.argtypes = [_i64, _i64, _i64, _i64, _i64, _p, _i32, _p, _p, _p]
    for suf in ("f", "d"):
        g = lambda name: getattr(L, f"orc{suf}_{name}")  # noqa: E731
        g("new").restype = _p
        g("new").argtypes = [_p, _i64, _i32, _i32, _f32, _f32, _p]
        g("free").argtypes = [_p]
        g("set_lr_schedule").restype = _i32
        g("set_lr_schedule").argtypes = [_p, _p, _p, _i32]
        g("set_lr_policy").restype = _i32
        g("set_lr_policy").argtypes = [_p, _i32, _f32]
        g("set_members").restype = _i32
        g("set_members").argtypes = [_p, _p, _i32]
        g("set_momentum_policy").restype = _i32
        g("set_momentum_policy").argtypes = [_p, _i32, _i64, _i64]
        g("set_nesterov").restype = _i32
        g("set_nesterov").argtypes = [_p, _i32]
        g("bsp_step").restype = _i32
        g("bsp_step").argtypes = [_p, _p, _p, _p, _i32]
        g("asp_push").restype = _i32
        g("asp_push").argtypes = [_p, _i32, _p, _i64, _p]
        g("pull").restype = _i32
        g("pull").argtypes = [_p, _i32, _p, _p]
        g("switch").restype = _i32
        g("switch").argtypes = [_p, _i32, _i64]
        g("read_params").restype = _i32
        g("read_params").argtypes = [_p, _p]
        g("read_velocity").restype = _i32
        g("read_velocity").argtypes = [_p, _p]
        g("stats").restype = _i32
        g("stats").argtypes = [_p, _p, _p, _p, _i32, _p]
        g("log_len").restype = _i64
        g("log_len").argtypes = [_p]
        g("log_get").restype = _i32
        g("log_get").argtypes = [_p, _i64, _p]
        g("current_lr").restype = _f32
        g("current_lr").argtypes = [_p, _i32]
    L.orc_splitmix64.restype = _u64
    L.orc_splitmix64.argtypes = [_u64]
    L.orc_synth_grad.argtypes = [_u64, _i32, _i64, _i64, _i64, _p]
    L.orc_schedule.restype = _i64
    L.orc_schedule.argtypes = [_i32, _p, _i64, _u64, _i32, _i64, _i64, _i64, _i64, _p, _p, _p]
    L.orc_softmax_loss_grad.restype = _f64
    L.orc_softmax_loss_grad.argtypes = [_p, _p, _i32, _i32, _i32, _p, _p]
    L.orc_detector_new.restype = _p
    L.orc_detector_new.argtypes = [_i32, _i32]
    L.orc_detector_free.argtypes = [_p]
    L.orc_detector_window.restype = _i32
    L.orc_detector_window.argtypes = [_p, _p, _p, _p]
    L.orc_detector_window_masked.restype = _i32
    L.orc_detector_window_masked.argtypes = [_p, _p, _p, _p, _p]
    _lib = L
    return L


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ---------------------------------------------------------------------------------------------------------------
# layout / lr / Table I
def shard_pad(P: int, S: int) -> int:
    return int(lib().orc_shard_pad(P, S))


def shard_offsets(P: int, S: int) -> np.ndarray:
    off = np.zeros(S + 1, dtype=np.int64)
    lib().orc_shard_offsets(P, S, _ptr(off))
    return off


def shard_owner(s: int, S: int, G: int) -> int:
    return int(lib().orc_shard_owner(s, S, G))


def worker_host(j: int, n: int, G: int) -> int:
    return int(lib().orc_worker_host(j, n, G))


def lr_factor(version: int, bounds, factors) -> float:
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    f = np.ascontiguousarray(factors, dtype=np.float32)
    return float(lib().orc_lr_factor(version, _ptr(b) if len(b) else None, _ptr(f) if len(f) else None, len(b)))


def lr(eta: float, factor: float, proto: int, n: int, asp_rule: int = 0) -> float:
    return float(lib().orc_lr(eta, factor, proto, n, asp_rule))


def table1(W: int, B: int, N: int, s_num: int, s_den: int, Wb):
    Wb = np.ascontiguousarray(Wb, dtype=np.int64)
    out = np.zeros(max(len(Wb), 1), dtype=np.int64)
    bsp = np.zeros(1, dtype=np.int64)
    asp = np.zeros(1, dtype=np.int64)
    rc = lib().orc_table1(W, B, N, s_num, s_den, _ptr(Wb) if len(Wb) else None, len(Wb), _ptr(bsp), _ptr(asp),
                          _ptr(out))
    if rc != 0:
        raise ValueError("Table I quantities are not integral")
    return int(bsp[0]), int(asp[0]), [int(x) for x in out[:len(Wb)]]


# ---------------------------------------------------------------------------------------------------------------
# state machine
class Oracle:
    """The BSP/ASP/switch state machine. ``dtype`` float32 (parity) or float64 (identities)."""

    def __init__(self, params, n_shards: int, n_workers: int, lr: float, momentum: float, dtype=np.float32):
        self.dtype = np.dtype(dtype)
        self._suf = "f" if self.dtype == np.float32 else "d"
        self._L = lib()
        p = np.ascontiguousarray(params, dtype=self.dtype)
        self.P = p.size
        self.n = n_workers
        st = np.zeros(1, dtype=np.int32)
        self._h = self._fn("new")(_ptr(p), p.size, n_shards, n_workers, lr, momentum, _ptr(st))
        self.status_init = int(st[0])
        if not self._h:
            raise ValueError(f"oracle init rejected: status {self.status_init}")

    def _fn(self, name):
        return getattr(self._L, f"orc{self._suf}_{name}")

    def close(self):
        if getattr(self, "_h", None):
            self._fn("free")(self._h)
            self._h = None

    __del__ = close

    def set_lr_schedule(self, bounds, factors) -> int:
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        f = np.ascontiguousarray(factors, dtype=np.float32)
        return int(self._fn("set_lr_schedule")(self._h, _ptr(b) if len(b) else None, _ptr(f) if len(f) else None,
                                               len(b)))

    def set_lr_policy(self, asp_rule: int, weight_decay: float) -> int:
        return int(self._fn("set_lr_policy")(self._h, asp_rule, weight_decay))

    def set_members(self, workers) -> int:
        w = np.ascontiguousarray(workers, dtype=np.int32)
        return int(self._fn("set_members")(self._h, _ptr(w), w.size))

    def set_nesterov(self, on: bool) -> int:
        return int(self._fn("set_nesterov")(self._h, int(on)))

    def set_momentum_policy(self, rule: int, samples_per_epoch: int = 1, batch: int = 1) -> int:
        return int(self._fn("set_momentum_policy")(self._h, rule, samples_per_epoch, batch))

    def bsp_step(self, grads, workers=None, versions=None) -> int:
        gs = [np.ascontiguousarray(g, dtype=self.dtype) for g in grads]
        if workers is None:
            workers = list(range(len(gs)))
        if versions is None:
            versions = [self.version] * len(gs)
        ptrs = (ctypes.c_void_p * len(gs))(*[_ptr(g) for g in gs])
        w = np.ascontiguousarray(workers, dtype=np.int32)
        v = np.ascontiguousarray(versions, dtype=np.int64)
        return int(self._fn("bsp_step")(self._h, ctypes.cast(ptrs, ctypes.c_void_p), _ptr(w), _ptr(v), len(gs)))

    def asp_push(self, worker: int, grad, version: int):
        g = np.ascontiguousarray(grad, dtype=self.dtype)
        st = np.zeros(1, dtype=np.int64)
        rc = int(self._fn("asp_push")(self._h, worker, _ptr(g), version, _ptr(st)))
        return rc, int(st[0])

    def pull(self, worker: int, want_params: bool = True):
        dst = np.empty(self.P, dtype=self.dtype) if want_params else None
        ver = np.zeros(1, dtype=np.int64)
        rc = int(self._fn("pull")(self._h, worker, _ptr(dst) if dst is not None else None, _ptr(ver)))
        return rc, dst, int(ver[0])

    def switch(self, protocol: int, at_step: int) -> int:
        return int(self._fn("switch")(self._h, protocol, at_step))

    def params(self) -> np.ndarray:
        dst = np.empty(self.P, dtype=self.dtype)
        self._fn("read_params")(self._h, _ptr(dst))
        return dst

    def velocity(self) -> np.ndarray:
        dst = np.empty(self.P, dtype=self.dtype)
        self._fn("read_velocity")(self._h, _ptr(dst))
        return dst

    def stats(self, hist_len: int = 64):
        ver = np.zeros(1, dtype=np.int64)
        proto = np.zeros(1, dtype=np.int32)
        hist = np.zeros(hist_len, dtype=np.uint64)
        dropped = np.zeros(1, dtype=np.uint64)
        rc = int(self._fn("stats")(self._h, _ptr(ver), _ptr(proto), _ptr(hist), hist_len, _ptr(dropped)))
        return dict(status=rc, version=int(ver[0]), protocol=int(proto[0]), hist=hist, dropped=int(dropped[0]))

    @property
    def version(self) -> int:
        return self.stats(1)["version"]

    def log(self) -> np.ndarray:
        n = int(self._fn("log_len")(self._h))
        out = np.zeros((n, 4), dtype=np.int64)
        rec = np.zeros(4, dtype=np.int64)
        for i in range(n):
            self._fn("log_get")(self._h, i, _ptr(rec))
            out[i] = rec
        return out

    def current_lr(self, protocol: int) -> float:
        return float(self._fn("current_lr")(self._h, protocol))


# ---------------------------------------------------------------------------------------------------------------
# synthetic inputs, toy model, detector
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def synth_grad(seed: int, j: int, k: int, i0: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float32)
    lib().orc_synth_grad(seed, j, k, i0, count, _ptr(out))
    return out


def schedule(n: int, period, n_push: int, jitter: int = 0, seed: int = 7, slow_worker: int = -1,
             slow_factor: int = 1, slow_t0: int = 0, slow_t1: int = 0):
    per = np.ascontiguousarray(period, dtype=np.int64)
    cap = 2 * n_push + n
    kind = np.zeros(cap, dtype=np.int32)
    worker = np.zeros(cap, dtype=np.int32)
    tick = np.zeros(cap, dtype=np.int64)
    e = lib().orc_schedule(n, _ptr(per), jitter, seed, slow_worker, slow_factor, slow_t0, slow_t1, n_push,
                           _ptr(kind), _ptr(worker), _ptr(tick))
    return kind[:e], worker[:e], tick[:e]


def softmax_loss_grad(X, y, W):
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    W = np.ascontiguousarray(W, dtype=np.float64)
    B, d = X.shape
    C = W.size // d
    grad = np.zeros(d * C, dtype=np.float64)
    loss = lib().orc_softmax_loss_grad(_ptr(X), _ptr(y), B, d, C, _ptr(W), _ptr(grad))
    return float(loss), grad


class Detector:
    def __init__(self, n: int, K: int = 3):
        self._L = lib()
        self.n = n
        self._h = self._L.orc_detector_new(n, K)

    def window(self, samples, busy, mask=None):
        """One detection window; `mask` (elastic policy): only workers with mask[k] != 0 are measured."""
        s = np.ascontiguousarray(samples, dtype=np.float64)
        b = np.ascontiguousarray(busy, dtype=np.float64)
        flag = np.zeros(self.n, dtype=np.int32)
        if mask is None:
            clean = self._L.orc_detector_window(self._h, _ptr(s), _ptr(b), _ptr(flag))
        else:
            m = np.ascontiguousarray(mask, dtype=np.uint8)
            clean = self._L.orc_detector_window_masked(self._h, _ptr(s), _ptr(b), _ptr(m), _ptr(flag))
        return flag.astype(bool), bool(clean)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_detector_free(self._h)
            self._h = None


# ---------------------------------------------------------------------------------------------------------------
# online straggler scenario (config 4)
SCENARIO_KEYS = ("n_workers", "batch", "total_samples", "quota_num", "quota_den", "period", "jitter", "sched_seed",
                 "grad_seed", "slow_worker", "slow_factor", "slow_t0", "slow_t1", "window_ticks", "K", "policy")


def scenario(sc: dict, state: "Oracle | None" = None, P: int = 0, cap: int = 256):
    """Runs the config-4 scenario on `state` (fp32 Oracle) or dry. Returns (switch log [(tick, version, to,
    reason, members)], result dict)."""
    L = lib()
    if not hasattr(L, "_scen"):
        L.orc_scenario_run.restype = _i64
        L.orc_scenario_run.argtypes = [_p, _i64, _i32, _i64, _i64, _i64, _i64, _i64, _i64, _u64, _u64, _i32, _i64,
                                       _i64, _i64, _i64, _i32, _i32, _p, _i32, _p]
        L._scen = True
    log = np.zeros((cap, 5), dtype=np.int64)
    res = np.zeros(7, dtype=np.int64)
    if state is not None:
        assert state.dtype == np.float32
    nsw = L.orc_scenario_run(state._h if state is not None else None, P, sc["n_workers"], sc["batch"],
                             sc["total_samples"], sc["quota_num"], sc["quota_den"], sc["period"], sc["jitter"],
                             sc["sched_seed"], sc["grad_seed"], sc["slow_worker"], sc["slow_factor"], sc["slow_t0"],
                             sc["slow_t1"], sc["window_ticks"], sc["K"], sc.get("policy", 0), _ptr(log), cap,
                             _ptr(res))
    keys = ("bsp_steps", "asp_pushes", "dropped", "end_tick", "version", "windows", "n_switches")
    return [tuple(int(x) for x in r) for r in log[:min(nsw, cap)]], dict(zip(keys, (int(x) for x in res)))


# ---------------------------------------------------------------------------------------------------------------
# dynamic switching criterion
def _crit_sigs(L):
    if not hasattr(L, "_crit"):
        L.orc_criterion.argtypes = [_p, _i32, _i64, _p, _p, _p]
        L.orc_softmax_per_sample.argtypes = [_p, _p, _i32, _i32, _i32, _p, _p]
        L.orc_criterion_observe.restype = _i32
        L.orc_criterion_observe.argtypes = [_p, _f64, _f64, _f64, _i32]
        L._crit = True
    return L


def criterion(per_sample, g_prev):
    """(|Delta|, sigma) from a B x P matrix of per-sample gradients and the lagged batch gradient."""
    L = _crit_sigs(lib())
    ps = np.ascontiguousarray(per_sample, dtype=np.float64)
    gp = np.ascontiguousarray(g_prev, dtype=np.float64)
    B, P = ps.shape
    nd = np.zeros(1)
    sg = np.zeros(1)
    L.orc_criterion(_ptr(ps), B, P, _ptr(gp), _ptr(nd), _ptr(sg))
    return float(nd[0]), float(sg[0])


def softmax_per_sample(X, y, W):
    L = _crit_sigs(lib())
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    W = np.ascontiguousarray(W, dtype=np.float64)
    B, d = X.shape
    C = W.size // d
    out = np.zeros((B, d * C))
    L.orc_softmax_per_sample(_ptr(X), _ptr(y), B, d, C, _ptr(W), _ptr(out))
    return out


class CriterionRule:
    def __init__(self, c: float = 2.0, T: int = 5):
        self.c, self.T = c, T
        self._run = np.zeros(1, dtype=np.int32)

    def observe(self, norm_delta: float, sigma: float) -> bool:
        return bool(_crit_sigs(lib()).orc_criterion_observe(_ptr(self._run), norm_delta, sigma, self.c, self.T))
