"""Config 4: the online straggler scenario (greedy policy P:1421 over the detector P:1425, transient <= 100 s P:1416).

CPU: the library's host-only dry run equals the oracle's, event for event; the oracle's run is pinned to the rules
(switch times bounded by the detection windows, workload preserved = Table I's step counts). GPU: the same scenario
through the C-ABI with real gradients equals the oracle bit-for-bit.
"""
import numpy as np
import pytest

BASE = dict(n_workers=8, batch=128, total_samples=64000 * 128, quota_num=1, quota_den=4, period=1000, jitter=0,
            sched_seed=7, grad_seed=20241018, slow_worker=7, slow_factor=4, slow_t0=20000, slow_t1=120000,
            window_ticks=10000, K=3, policy=0)


@pytest.fixture(scope="module")
def ss():
    from paper_2104_08364_b200 import build
    build.build()
    from paper_2104_08364_b200 import syncswitch
    return syncswitch


CASES = [
    BASE,
    dict(BASE, jitter=100),
    dict(BASE, slow_worker=-1),
    dict(BASE, quota_num=1, quota_den=2, slow_t0=300000, slow_t1=380000),
    dict(BASE, n_workers=4, slow_worker=2, total_samples=8000 * 128, quota_num=1, quota_den=2, slow_t0=0,
         slow_t1=50000, K=2, window_ticks=5000),
    dict(BASE, quota_num=0, quota_den=1),
    dict(BASE, quota_num=1, quota_den=1, total_samples=2000 * 128 * 8),
    dict(BASE, policy=1),
    dict(BASE, policy=1, jitter=100),
    dict(BASE, policy=1, n_workers=4, slow_worker=2, total_samples=8000 * 128, quota_num=1, quota_den=2, K=2,
         window_ticks=5000, slow_t0=0, slow_t1=50000),
    dict(BASE, policy=2),
]


@pytest.mark.parametrize("sc", CASES)
def test_dry_run_matches_oracle(ss, orc, sc):
    s, log_a, res_a = ss.ss_scenario_run(None, sc)
    log_b, res_b = orc.scenario(sc)
    assert s == 0 and log_a == log_b and res_a == res_b


@pytest.mark.parametrize("split", [(5, 95), (10, 90), (25, 75), (50, 50)])
def test_no_straggler_preserves_table1(orc, split):
    # no straggler, no jitter: only the timing-policy switch, and the step counts are Table I's
    sc = dict(BASE, slow_worker=-1, quota_num=split[0], quota_den=100)
    log, res = orc.scenario(sc)
    bsp, asp, _ = orc.table1(64000 * 128, 128, 8, split[0], 100, [])
    assert (res["bsp_steps"], res["asp_pushes"]) == (bsp, asp)
    assert log == [(bsp * 1000, bsp, 1, 0, 8)]       # switch to ASP once, at version = BSP steps
    assert res["dropped"] == 0 and res["version"] == bsp + asp


def test_greedy_switches_bounded_by_windows(orc):
    # Straggler transient [t0, t1) starting during BSP: the greedy policy switches to ASP once the detector has seen K
    # flagged windows, and back to BSP K clean windows after the transient ends; in-flight pushes are dropped; the
    # BSP quota and the total workload are still exactly met (Table I's 25-75 row: 2000 + 48000).
    sc = BASE
    log, res = orc.scenario(sc)
    T, D, K, t0, t1 = sc["period"], sc["window_ticks"], sc["K"], sc["slow_t0"], sc["slow_t1"]
    assert [(to, why) for _, _, to, why, _ in log] == [(1, 1), (0, 2), (1, 0)]
    assert t0 + K * D <= log[0][0] <= t0 + (K + 1) * D + 4 * T
    assert t1 + K * D <= log[1][0] <= t1 + (K + 1) * D + 4 * T
    assert res["dropped"] == sc["n_workers"]
    assert (res["bsp_steps"], res["asp_pushes"]) == (2000, 48000)
    assert res["version"] == 2000 + 48000


def test_elastic_policy_rules(orc):
    # the detected straggler leaves the BSP barrier (K flagged windows into the transient), BSP continues
    # with n - 1 workers until the BSP quota is met, then all n are restored and ASP runs the rest: one protocol
    # switch in total, no dropped pushes.
    sc = dict(BASE, policy=1)
    log, res = orc.scenario(sc)
    T, D, K, t0 = sc["period"], sc["window_ticks"], sc["K"], sc["slow_t0"]
    assert [(to, why, m) for _, _, to, why, m in log] == [(0, 3, 7), (1, 0, 8)]
    assert t0 + K * D <= log[0][0] <= t0 + (K + 1) * D + 4 * T
    assert res["dropped"] == 0
    quota = sc["total_samples"] * sc["quota_num"] // sc["quota_den"]
    removal_version = log[0][1]
    bsp_samples = removal_version * 8 * 128 + (res["bsp_steps"] - removal_version) * 7 * 128
    assert bsp_samples >= quota and bsp_samples - 7 * 128 < quota          # the quota is met exactly once
    assert res["asp_pushes"] * 128 + bsp_samples >= sc["total_samples"]
    # A straggler that stays slow through the BSP phase holds every BSP superstep to 4000 ticks unless removed: then
    # the elastic run finishes first. (A short transient can favour no policy, because the removed worker stays out
    # until the quota is met, by design.)
    persistent = dict(sc, slow_t1=10 ** 12)
    assert orc.scenario(persistent)[1]["end_tick"] < orc.scenario(dict(persistent, policy=2))[1]["end_tick"]


def test_elastic_bsp_equals_smaller_cluster(orc):
    # BSP over m of n workers == BSP of an m-worker cluster (configuration policy re-derived for m)
    rng = np.random.default_rng(31)
    P, n = 257, 6
    members = [0, 2, 3, 5]
    w0 = rng.standard_normal(P).astype(np.float32)
    gs = [[rng.standard_normal(P).astype(np.float32) for _ in range(n)] for _ in range(3)]
    a = orc.Oracle(w0, 3, n, 0.05, 0.9)
    assert a.set_members(members) == 0
    b = orc.Oracle(w0, 3, len(members), 0.05, 0.9)
    for r in range(3):
        assert a.bsp_step([gs[r][j] for j in members], workers=members) == 0
        assert b.bsp_step([gs[r][j] for j in members]) == 0
    assert np.array_equal(a.params(), b.params()) and np.array_equal(a.velocity(), b.velocity())
    assert a.bsp_step([gs[0][j] for j in range(n)]) == 3          # a removed worker at the barrier: SS_E_PROTOCOL
    assert a.set_members([0, 0]) == 1 and a.set_members([]) == 1 and a.set_members([6]) == 1


def test_quota_edge_cases(orc):
    # a zero BSP quota: the run starts with BSP, whose first superstep already meets the quota
    log, res = orc.scenario(dict(BASE, quota_num=0, quota_den=1))
    assert res["bsp_steps"] == 1 and log[0][3] == 0
    log, res = orc.scenario(dict(BASE, quota_num=1, quota_den=1, slow_worker=-1, total_samples=100 * 1024))
    assert res["asp_pushes"] == 0 and res["bsp_steps"] == 100              # pure BSP


@pytest.mark.gpu
@pytest.mark.parametrize("sc", [dict(BASE, total_samples=4000 * 128, quota_num=1, quota_den=2, slow_t0=10000,
                                     slow_t1=60000),
                                dict(BASE, n_workers=4, slow_worker=1, total_samples=3000 * 128, quota_num=1,
                                     quota_den=3, slow_t0=5000, slow_t1=40000, K=2, window_ticks=6000, jitter=50)])
def test_scenario_on_gpu_bit_exact(ss, orc, sc):
    _scenario_on_gpu(ss, orc, sc)


@pytest.mark.gpu
def test_elastic_scenario_on_gpu_bit_exact(ss, orc):
    _scenario_on_gpu(ss, orc, dict(BASE, policy=1, total_samples=4000 * 128, quota_num=1, quota_den=2,
                                   slow_t0=10000, slow_t1=60000))


@pytest.mark.gpu
def test_scenario_on_gpu_config2_shape(ss, orc):
    """The straggler scenario at the ResNet-32 shape (P = 464,154, n = S = 8: SV §8(d) config 4 "or 464,154"), a
    shortened workload that still detects the straggler, switches to ASP and back: bit-exact with the oracle."""
    _scenario_on_gpu(ss, orc, dict(BASE, total_samples=1200 * 128, quota_num=1, quota_den=2, slow_t0=5000,
                                   slow_t1=45000), P=464154, S=8)


def _scenario_on_gpu(ss, orc, sc, P=4099, S=4):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = sc["n_workers"]
    w0 = orc.synth_grad(20241019, 255, 0, 0, P) * np.float32(64.0)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    s, log_g, res_g = ss.ss_scenario_run(g.ctx, sc)
    assert s == 0, g.last_error()
    log_o, res_o = orc.scenario(sc, o, P)
    assert log_g == log_o and res_g == res_o
    g.sync()
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    sg, so = g.stats(64), o.stats(64)
    assert sg["version"] == so["version"] and np.array_equal(sg["hist"], so["hist"])
    assert sg["dropped"] == so["dropped"] == res_o["dropped"]
    g.close()
