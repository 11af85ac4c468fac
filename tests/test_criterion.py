"""Dynamic switching criterion: pins for the oracle (CPU) and parity of the
CUDA kernel (ss_dynamic_criterion) against it (GPU)."""
import numpy as np
import pytest

from conftest import golden


def test_worked_example(orc):
    (a, b, gp, nd, sg, c, sat), = [list(map(float, r)) for r in golden("criterion_1d.txt")]
    got_nd, got_sg = orc.criterion(np.array([[a], [b]]), np.array([gp]))
    assert got_nd == pytest.approx(nd, rel=1e-12) and got_sg == pytest.approx(sg, rel=1e-12)
    assert (got_nd < c * got_sg) == bool(sat)


def test_identical_samples_have_zero_sigma(orc):
    # per-sample gradients all equal to g -> sigma = 0 (never satisfied for |Delta| > 0)
    rng = np.random.default_rng(0)
    row = rng.standard_normal(50)
    nd, sg = orc.criterion(np.tile(row, (6, 1)), row + 0.01)
    assert nd > 0 and sg <= 1e-12 * nd            # zero up to the rounding of the mean
    rule = orc.CriterionRule(c=2.0, T=1)
    assert not rule.observe(nd, sg)


def _per_sample(rng, B=8, P=40):
    return rng.standard_normal((B, P))


def test_scale_invariance_and_bounds(orc):
    rng = np.random.default_rng(1)
    ps = _per_sample(rng)
    g = ps.mean(axis=0)
    delta = rng.standard_normal(ps.shape[1])
    nd1, s1 = orc.criterion(ps, g - delta)
    nd2, s2 = orc.criterion(ps, g - 3.5 * delta)
    assert nd2 == pytest.approx(3.5 * nd1, rel=1e-12) and s2 == pytest.approx(s1, rel=1e-12)  # sigma is per unit |Delta|
    # Cauchy-Schwarz: sigma <= sqrt(sum_b |grad_b - g|^2) / B
    assert s1 <= np.sqrt(((ps - g) ** 2).sum()) / ps.shape[0] + 1e-15


def test_coordinate_direction_is_standard_error(orc):
    # Delta along coordinate m: sigma = population std of that coordinate / sqrt(B) (the paper's "sample standard
    # deviation" of the batch-gradient noise in the direction Delta)
    rng = np.random.default_rng(2)
    ps = _per_sample(rng, B=16)
    g = ps.mean(axis=0)
    for m in (0, 7, 39):
        e = np.zeros(ps.shape[1])
        e[m] = 0.25
        nd, sg = orc.criterion(ps, g - e)
        assert nd == pytest.approx(0.25, rel=1e-12)
        assert sg == pytest.approx(np.std(ps[:, m]) / np.sqrt(16), rel=1e-10)


def test_softmax_per_sample_mean_is_the_batch_gradient(orc):
    from inputs import toy_dataset
    X, y = toy_dataset(seed=3, n_points=12, d=17, C=4)
    W = np.random.default_rng(3).standard_normal(17 * 4) * 0.2
    ps = orc.softmax_per_sample(X, y, W)
    _, g = orc.softmax_loss_grad(X, y, W)
    np.testing.assert_allclose(ps.mean(axis=0), g, rtol=1e-12, atol=1e-15)
    # rank one: grad_b = x_b (x) r_b
    for b in range(3):
        M = ps[b].reshape(17, 4)
        assert np.linalg.matrix_rank(M, tol=1e-10) <= 1


def test_persistence_rule(orc, ss_lib):
    # T = 3 with only 2 consecutive satisfactions does not fire; the third does
    for rule in (orc.CriterionRule(c=2.0, T=3), ss_lib.CriterionRule(c=2.0, T=3)):
        seq = [(0.1, 1.0), (0.1, 1.0), (5.0, 1.0), (0.1, 1.0), (0.1, 1.0), (0.0, 0.0)]
        assert [rule.observe(a, b) for a, b in seq] == [False, False, False, False, False, True]
    rng = np.random.default_rng(4)
    a_rule, b_rule = orc.CriterionRule(c=1.5, T=2), ss_lib.CriterionRule(c=1.5, T=2)
    for _ in range(300):
        nd, sg = float(np.float32(rng.random())), float(np.float32(rng.random()))
        assert a_rule.observe(nd, sg) == b_rule.observe(nd, sg)


@pytest.fixture(scope="module")
def ss_lib():
    from paper_2104_08364_b200 import build
    build.build()
    from paper_2104_08364_b200 import syncswitch
    return syncswitch


@pytest.mark.gpu
def test_criterion_kernel_parity(orc, ss_lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from inputs import toy_dataset
    X, y = toy_dataset(seed=1, n_points=64)
    B, d, C = 16, X.shape[1], 8
    rng = np.random.default_rng(5)
    for trial in range(4):
        W = (rng.standard_normal(d * C) * 0.02).astype(np.float32)
        idx, idx_prev = rng.choice(64, B, replace=False), rng.choice(64, B, replace=False)
        _, gp = orc.softmax_loss_grad(X[idx_prev], y[idx_prev], W.astype(np.float64))
        ps = orc.softmax_per_sample(X[idx], y[idx], W.astype(np.float64))
        nd_o, sg_o = orc.criterion(ps, gp)
        Xd, yd = torch.from_numpy(X[idx]).cuda(), torch.from_numpy(y[idx]).cuda()
        g_out = torch.empty(d * C, device="cuda")
        stats = torch.empty(2, device="cuda")
        gpd = torch.from_numpy(gp.astype(np.float32)).cuda()
        assert ss_lib.ss_dynamic_criterion(Xd, yd, B, d, C, torch.from_numpy(W).cuda(), gpd, g_out, stats) == 0
        nd_g, sg_g = stats.cpu().numpy().astype(np.float64)
        # the kernel reads fp32 gradients: tolerance derived from fp32 rounding of g and g_prev (~1e-7 relative)
        assert nd_g == pytest.approx(nd_o, rel=1e-5) and sg_g == pytest.approx(sg_o, rel=1e-4)
        np.testing.assert_allclose(g_out.cpu().numpy(), ps.mean(axis=0), rtol=1e-5, atol=1e-7)


@pytest.mark.gpu
def test_toy_dynamic_switch(orc, ss_lib):
    """Config-1 toy model under BSP with the dynamic criterion deciding the switch: every superstep the
    criterion kernel runs on worker 0's batch against worker 0's previous-step batch gradient (k = 1); after T
    satisfied steps ss_switch(ASP) is issued. The oracle evaluates the same quantities at the same parameters."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from inputs import minibatch_order, toy_dataset
    ss = ss_lib
    n, S, B, d, C = 2, 2, 16, 1024, 8
    X, y = toy_dataset(seed=1, mean_scale=0.05)     # overlapping classes: the batch-gradient noise persists
    order = minibatch_order(1, len(X), 2 * 200, B)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    P = d * C
    g = ss.SyncSwitch(torch.zeros(P, device="cuda"), S, n, 0.1, 0.9)
    rule_g, rule_o = ss.CriterionRule(c=6.0, T=3), orc.CriterionRule(c=6.0, T=3)
    W = torch.empty(P, device="cuda")
    g_prev = torch.zeros(P, device="cuda")
    stats = torch.empty(2, device="cuda")
    loss = torch.empty(1, device="cuda")
    fired_at = None
    gp_host = np.zeros(P)
    for step in range(200):
        g.pull(0, W)
        g.sync()
        bi = [torch.from_numpy(order[2 * step + j]).cuda() for j in range(n)]
        g0 = torch.empty(P, device="cuda")
        assert ss.ss_dynamic_criterion(Xd[bi[0]].contiguous(), yd[bi[0]].contiguous(), B, d, C, W, g_prev, g0,
                                       stats) == 0
        g1 = torch.empty(P, device="cuda")
        assert ss.ss_softmax_grad(Xd[bi[1]].contiguous(), yd[bi[1]].contiguous(), B, d, C, W, g1, loss) == 0
        nd, sg = (float(x) for x in stats.cpu().numpy())
        Wh = W.cpu().numpy().astype(np.float64)
        ps = orc.softmax_per_sample(X[order[2 * step]], y[order[2 * step]], Wh)
        nd_o, sg_o = orc.criterion(ps, gp_host) if step > 0 else orc.criterion(ps, np.zeros(P))
        # Delta = g - g_prev inherits the fp32 rounding of the kernel's gradients (logits summed over d = 1024 in
        # fp32, relative error ~1e-5 per probability): the tolerance is relative to the gradient scale |g| + |g_prev|
        scale = np.linalg.norm(ps.mean(axis=0)) + np.linalg.norm(gp_host)
        assert abs(nd - nd_o) <= 1e-4 * nd_o + 1e-4 * scale
        assert abs(sg - sg_o) <= 1e-3 * sg_o + 1e-4 * scale
        fire_g, fire_o = rule_g.observe(nd, sg), rule_o.observe(nd_o, sg_o)
        if abs(nd_o - 6.0 * sg_o) > 0.05 * nd_o + 1e-4 * scale:   # away from the threshold both decide alike
            assert fire_g == fire_o
        gp_host = ps.mean(axis=0)
        g_prev = g0.clone()
        g.bsp_step([g0, g1])
        if fire_g:
            fired_at = step
            g.switch(ss.SS_ASP, 0)
            break
    assert fired_at is not None, "the criterion never fired"
    assert g.stats()["protocol"] == ss.SS_ASP and g.version == fired_at + 1
    g.close()
