"""bench.py --workload host logic (CPU): the ASP arrival order with the versions each worker sends, checked against the
oracle's state machine, and the Table I step counts of the whole-workload runs."""
import numpy as np
import pytest

import bench
import oracle as orc
from paper_2104_08364_b200 import syncswitch as ss


def test_round_robin_staleness_closed_form():
    # equal periods, no jitter: the first round's pushes all carry version 0 (staleness 0..n-1, ties by worker id),
    # afterwards every worker's push has exactly n-1 other pushes since its pull (steady state)
    n, n_push = 8, 80
    kind, worker, version = bench.asp_workload_events(n, n_push, 0, jitter=0)
    assert kind.size == n + 2 * n_push and (kind[:n] == 1).all()
    ver, stale = 0, []
    for k, v in zip(kind, version):
        if k == 0:
            stale.append(ver - int(v))
            ver += 1
    assert stale[:n] == list(range(n)) and set(stale[n:]) == {n - 1}


def test_jittered_events_accepted_by_oracle():
    orc.build()
    n, P, n_bsp, n_push = 8, 64, 5, 300
    w0 = np.linspace(-1, 1, P, dtype=np.float32)
    o = orc.Oracle(w0, 2, n, 0.1, 0.9)
    g = np.full(P, 1 / 128, dtype=np.float32)
    for t in range(n_bsp):
        assert o.bsp_step([g] * n, versions=[t] * n) == 0
    assert o.switch(orc.ASP, 0) == 0
    kind, worker, version = bench.asp_workload_events(n, n_push, n_bsp, jitter=100)
    hist = {}
    for k, j, v in zip(kind, worker, version):
        if k == 0:
            rc, st = o.asp_push(int(j), g, int(v))
            assert rc == 0
            assert st == o.version - 1 - int(v)
            hist[st] = hist.get(st, 0) + 1
        else:
            rc, _, pv = o.pull(int(j), want_params=False)
            assert rc == 0 and pv == int(v)
    assert o.version == n_bsp + n_push
    assert max(hist) > n - 1          # jitter reorders arrivals: some pushes are staler than the steady state


# W_i -> W_i/B - W s/B + W s/(B n): config 2 (s = 1/16) 32000 - 4000 + 500, config 3 (s = 1/8) 32000 - 8000 + 1000
@pytest.mark.parametrize("config,expect", [("2", (500, 60000, [28500, 44500])),
                                          ("3", (1000, 56000, [25000, 41000]))])
def test_workload_table1_counts(config, expect):
    wl = bench.WORKLOADS[config]
    s, got = ss.ss_table1(wl["W"], wl["B"], 8, *wl["s"], wl["Wb"])
    assert s == 0 and got == expect
    s, (b, a, bounds) = ss.ss_table1(wl["W"], wl["B"], 8, 1, 1, wl["Wb"])      # pure BSP
    assert s == 0 and (b, a, bounds) == (8000, 0, [4000, 6000])
    s, (b, a, bounds) = ss.ss_table1(wl["W"], wl["B"], 8, 0, 1, wl["Wb"])      # pure ASP
    assert s == 0 and (b, a, bounds) == (0, 64000, [32000, 48000])
