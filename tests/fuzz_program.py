"""Seeded random call programs for the protocol fuzz tests (tests/test_gpu_fuzz.py, tests/dist_fuzz_worker.py).

Holds none of the method's arithmetic: it only draws a shape, the per-context settings and a sequence of C-ABI calls.
Each side (the CUDA path, the oracle) asks it for the next call given ITS OWN protocol state (protocol, version, the
workers' last pull versions), so the two programs are identical exactly as long as the two implementations agree on
every protocol integer — which is what the tests check call by call.

Ops: ("bsp", bad) — a superstep of every worker at the current version (bad: 0 valid, 1 one worker missing,
2 one stale base version; errors only at world 1, where they stay rank-local); ("push", j, version);
("pull", j, want_snapshot) (at G > 1 the hosting rank always passes a destination — every pull moves data
there — and keeps the snapshot only when wanted); ("switch", protocol, at_step); ("check",) — sync and compare state.
"""
import numpy as np

BSP, ASP = 0, 1


class Program:
    def __init__(self, case_seed: int, world: int = 1):
        rng = np.random.default_rng(case_seed)
        self.rng = rng
        self.world = world
        self.n = int(rng.integers(1, 9))
        self.S = int(rng.integers(1, 9))
        if world > 1:                                 # shards are split evenly over the ranks (ss_init_dist)
            self.S = world * max(1, self.S // world)
        self.P = int(rng.choice([1, 3, 33, 1000, 4099, 20011, 70003]))
        self.window = int(rng.choice([1, 2, 5, 16, 64]))
        self.lam = float(rng.choice([0.0, 0.0, 1e-4]))
        self.asp_rule = int(rng.integers(0, 3))
        self.nesterov = bool(rng.integers(0, 4) == 0)
        self.bounds = sorted(int(b) for b in rng.choice(np.arange(1, 60), size=2, replace=False))
        self.factors = [0.1, 0.01]
        self.fused = int(rng.integers(0, 4)) if world > 1 else -1
        self.n_ops = int(rng.integers(20, 80))

    def next_op(self, protocol: int, version: int, base: dict):
        rng = self.rng
        # op mix by protocol (BSP: mostly supersteps; ASP: mostly pushes; the other protocol's call is an error)
        cut = (0.45, 0.55, 0.80, 0.95) if protocol == BSP else (0.08, 0.60, 0.85, 0.95)
        r = rng.random()
        if r < cut[0]:
            kind = rng.random()
            bad = 0
            if self.world == 1 and kind < 0.1 and self.n > 1:
                bad = 1
            elif self.world == 1 and kind < 0.2:
                bad = 2
            return ("bsp", bad, int(rng.integers(0, self.n)))
        if r < cut[1]:
            j = int(rng.integers(0, self.n))
            b = base.get(j, 0)
            if rng.random() < 0.05:
                b = version + 1                       # from the future -> SS_E_CAUSALITY
            return ("push", j, b)
        if r < cut[2]:
            return ("pull", int(rng.integers(0, self.n)), bool(rng.random() < 0.8))
        if r < cut[3]:
            return ("switch", int(rng.integers(0, 2)), version + int(rng.integers(-2, 6)))
        return ("check",)

    def bsp_call(self, op, version: int, workers):
        """(workers, versions) of a ("bsp", bad, which) op over the given (hosted) workers."""
        _, bad, which = op
        js = list(workers)
        vers = [version] * len(js)
        if bad == 1:
            js, vers = js[:-1], vers[:-1]             # missing worker -> SS_E_PROTOCOL
        elif bad == 2 and js:
            vers[which % len(js)] = version - 1       # stale base -> SS_E_BARRIER
        return js, vers
