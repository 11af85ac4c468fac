"""Pins for the CPU oracle (oracle/), against what the paper and the mathematics fix — never against itself.

Each test names the passage (P:L = PAPER.md line) or the closed form / brute force it uses. CPU only.
"""
import collections
import math

import numpy as np
import pytest

from conftest import golden

BSP, ASP = 0, 1


# ---------------------------------------------------------------------------------------------------------------
# Table I, lr schedule, config policy
def test_table1_all_rows(orc):
    W, B, N = 64000 * 128, 128, 8
    for row in golden("table1.txt"):
        sb, sa, bsp, asp, total, b1, b2 = map(int, row)
        got = orc.table1(W, B, N, sb, 100, [32000 * 128, 48000 * 128])
        assert got == (bsp, asp, [b1, b2]), row
        assert got[0] + got[1] == total


def test_table1_config2(orc):
    # SURVEY config 2: s = 6.25% of 64K -> 500 BSP + 60,000 ASP, boundaries [28,500, 44,500]
    assert orc.table1(64000 * 128, 128, 8, 1, 16, [32000 * 128, 48000 * 128]) == (500, 60000, [28500, 44500])


def test_lr_at_paper_values(orc):
    # P:1600 "learning rate to be 0.1 and decays ... at 32K and 48K steps with scaling factors of 0.1 and 0.01"
    b, f = [32000, 48000], [0.1, 0.01]
    for step, want in [(0, 0.1), (31999, 0.1), (32000, 0.01), (47999, 0.01), (48000, 0.001), (63999, 0.001)]:
        lr = orc.lr(0.1, orc.lr_factor(step, b, f), ASP, 1, 2)
        assert lr == pytest.approx(want, rel=1e-6), step


def test_lr_schedule_in_the_state_machine(orc):
    # P:1600 step decay applied by the protocol state: the factor is looked up at the PRE-increment version (reading
    # C9) and is right-continuous at a boundary. n = 1, mu = 0, unit gradients, w0 = 0: w_k = -sum of the lrs used.
    o = orc.Oracle([0.0], 1, 1, 0.1, 0.0, dtype=np.float64)
    assert o.set_lr_schedule([2, 4], [0.5, 0.25]) == 0
    eta = float(np.float32(0.1))
    lrs = [float(np.float32(eta * f)) for f in (1, 1, 0.5, 0.5, 0.25)]
    w = 0.0
    for k in range(5):
        assert o.current_lr(BSP) == pytest.approx(lrs[k], rel=1e-7)
        assert o.bsp_step([[1.0]]) == 0
        w -= lrs[k]
        assert o.params()[0] == pytest.approx(w, rel=1e-12), k
    # the same schedule under ASP (eta/sqrt(n) = eta at n = 1), continuing the version count
    o.switch(ASP, 0)
    assert o.asp_push(0, [1.0], o.version) == (0, 0)
    assert o.params()[0] == pytest.approx(w - lrs[4], rel=1e-12)


def test_config_policy_values(orc):
    # BSP lr = n*eta (linear scaling); ASP lr = eta/sqrt(n); n = 8, eta = 0.1
    assert orc.lr(0.1, 1.0, BSP, 8) == np.float32(0.8)
    assert orc.lr(0.1, 1.0, ASP, 8, 0) == np.float32(np.float64(np.float32(0.1)) / math.sqrt(8))
    assert orc.lr(0.1, 1.0, ASP, 8, 0) == pytest.approx(0.035355339, rel=1e-7)
    assert orc.lr(0.1, 1.0, ASP, 8, 1) == pytest.approx(0.0125, rel=1e-7)
    # n = 1 is the identity for every rule
    for proto, rule in [(BSP, 0), (ASP, 0), (ASP, 1), (ASP, 2)]:
        assert orc.lr(0.1, 1.0, proto, 1, rule) == np.float32(0.1)


# ---------------------------------------------------------------------------------------------------------------
# shard layout
@pytest.mark.parametrize("P,S,pad,ppad", [(464154, 8, 58048, 464384), (25557032, 8, 3194656, 25557248),
                                          (8192, 2, 4096, 8192), (1, 1, 32, 32), (100, 7, 32, 224)])
def test_shard_layout(orc, P, S, pad, ppad):
    assert orc.shard_pad(P, S) == pad and pad * S == ppad
    off = orc.shard_offsets(P, S)
    assert off[0] == 0 and off[-1] == P
    assert np.all(np.diff(off) >= 0)                       # disjoint, covering, in order
    assert all((o * 4) % 128 == 0 for o in off[:-1] if o < P)   # every shard starts 128-B aligned
    assert all(orc.shard_owner(s, S, 1) == 0 for s in range(S))
    # owners contiguous and balanced when G divides S
    for G in (1, 2, 4, 8):
        if S % G == 0:
            owners = [orc.shard_owner(s, S, G) for s in range(S)]
            assert owners == sorted(owners) and collections.Counter(owners) == {g: S // G for g in range(G)}


def test_worker_host_hand_cases(orc):
    # P:1071 (one PS per worker node) and SURVEY §8(a) a1: worker j runs on GPU floor(j*G/n) -- hand-enumerated cases
    cases = {
        (8, 1): [0] * 8,
        (8, 2): [0, 0, 0, 0, 1, 1, 1, 1],
        (8, 4): [0, 0, 1, 1, 2, 2, 3, 3],
        (8, 8): [0, 1, 2, 3, 4, 5, 6, 7],          # the paper's one worker per node
        (3, 2): [0, 0, 1],                         # floor(0)=0, floor(2/3)=0, floor(4/3)=1
        (2, 4): [0, 2],                            # more GPUs than workers: GPUs 1 and 3 host nobody
        (5, 3): [0, 0, 1, 1, 2],                   # floor(0, .6, 1.2, 1.8, 2.4)
    }
    for (n, G), want in cases.items():
        assert [orc.worker_host(j, n, G) for j in range(n)] == want, (n, G)
    # every GPU hosts floor(n/G) or ceil(n/G) workers, in contiguous ascending blocks, when n >= G
    for n in range(1, 40):
        for G in (1, 2, 3, 4, 8):
            h = [orc.worker_host(j, n, G) for j in range(n)]
            assert h == sorted(h) and all(0 <= x < G for x in h)
            if n >= G:
                assert set(collections.Counter(h).values()) <= {n // G, -(-n // G)}


# ---------------------------------------------------------------------------------------------------------------
# the paper's worked ASP example and BSP on the same gradients
def _asp_rows():
    return [r for r in golden("asp_trace.txt") if r[0] != "BSP"]


@pytest.mark.parametrize("row", _asp_rows())
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_asp_worked_trace(orc, row, dtype):
    w0, eta, lam, g11, g12, mu, w1, w1p, vfin, st1, st2 = map(float, row)
    o = orc.Oracle([w0], 1, 2, eta, mu, dtype=dtype)
    assert o.set_lr_policy(2, lam) == 0          # unscaled ASP lr: eta_t = eta exactly as in the equation
    assert o.switch(ASP, 0) == 0
    rc, _, v0 = o.pull(0)
    rc, _, v1 = o.pull(1)
    assert (v0, v1) == (0, 0)
    rc, s = o.asp_push(0, [g11], 0)
    assert rc == 0 and s == st1 and o.params()[0] == w1
    rc, s = o.asp_push(1, [g12], 0)              # computed at w0: stale by one update
    assert rc == 0 and s == st2 and o.params()[0] == w1p
    assert o.velocity()[0] == vfin


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_bsp_worked_example(orc, dtype):
    (_, w0, eta, lam, g11, g12, mu, w, v), = [r for r in golden("asp_trace.txt") if r[0] == "BSP"]
    o = orc.Oracle([float(w0)], 1, 2, float(eta), float(mu), dtype=dtype)
    o.set_lr_policy(0, float(lam))
    assert o.bsp_step([[float(g11)], [float(g12)]]) == 0
    assert o.params()[0] == float(w) and o.velocity()[0] == float(v)
    assert o.version == 1


# ---------------------------------------------------------------------------------------------------------------
# momentum step: special cases and the 1-D quadratic closed form
def test_momentum_special_cases(orc):
    rng = np.random.default_rng(1)
    w0 = rng.standard_normal(257).astype(np.float32)
    g = rng.standard_normal(257).astype(np.float32)
    # mu = 0: w' = w - eta*g, a single rounding (fma with v = g)
    o = orc.Oracle(w0, 3, 1, 0.25, 0.0)
    o.bsp_step([g])
    assert np.array_equal(o.params(), (w0.astype(np.float64) - 0.25 * g.astype(np.float64)).astype(np.float32))
    # g = 0 after one step: w'' = w' - eta*mu*v  (double mode, exact to rounding of the products)
    o = orc.Oracle(w0, 3, 1, 0.25, 0.5, dtype=np.float64)
    o.bsp_step([g])
    w1, v1 = o.params(), o.velocity()
    o.bsp_step([np.zeros(257)])
    np.testing.assert_allclose(o.params(), w1 - 0.25 * 0.5 * v1, rtol=0, atol=1e-15)


def test_momentum_quadratic_closed_form(orc):
    # L(x) = a x^2 / 2, g = a x. The state (v, x) evolves linearly: [v', x'] = M [v, x] with
    # M = [[mu, a], [-eta*mu, 1 - eta*a]]; x_t is read off M^t, an independent closed form.
    a, eta, mu, x0 = 0.75, 0.125, float(np.float32(0.9)), 2.0   # mu travels as fp32 through the API
    o = orc.Oracle([x0], 1, 1, eta, mu, dtype=np.float64)
    xs = []
    for _ in range(50):
        x = o.params()[0]
        assert o.bsp_step([[a * x]]) == 0
        xs.append(o.params()[0])
    M = np.array([[mu, a], [-eta * mu, 1 - eta * a]])
    for t in range(1, 51):
        want = (np.linalg.matrix_power(M, t) @ np.array([0.0, x0]))[1]
        assert xs[t - 1] == pytest.approx(want, rel=1e-12, abs=1e-14)


def test_nesterov_quadratic_closed_form(orc):
    # Nesterov (reading C28): v' = mu v + g, x' = x - eta (g + mu v'). On L = a x^2 / 2 (g = a x) the state is linear:
    # [v', x'] = N [v, x], N = [[mu, a], [-eta mu^2, 1 - eta a (1 + mu)]] (substitute v' into the x update).
    a, eta, mu, x0 = 0.75, 0.125, float(np.float32(0.9)), 2.0
    o = orc.Oracle([x0], 1, 1, eta, mu, dtype=np.float64)
    assert o.set_nesterov(True) == 0
    xs = []
    for _ in range(50):
        x = o.params()[0]
        assert o.bsp_step([[a * x]]) == 0
        xs.append(o.params()[0])
    N = np.array([[mu, a], [-eta * mu * mu, 1 - eta * a * (1 + mu)]])
    for t in range(1, 51):
        want = (np.linalg.matrix_power(N, t) @ np.array([0.0, x0]))[1]
        assert xs[t - 1] == pytest.approx(want, rel=1e-12, abs=1e-14)
    # the ASP push path applies the same step
    o = orc.Oracle([x0], 1, 1, eta, mu, dtype=np.float64)
    assert o.set_lr_policy(2, 0.0) == 0       # eta_ASP = eta
    o.set_nesterov(True)
    o.switch(orc.ASP, 0)
    v, x = 0.0, x0
    for t in range(20):
        rc, _ = o.asp_push(0, [a * o.params()[0]], t)
        assert rc == 0
        v, x = N @ np.array([v, x])
        assert o.params()[0] == pytest.approx(x, rel=1e-12, abs=1e-14)


def test_nesterov_special_cases(orc):
    rng = np.random.default_rng(4)
    w0 = rng.standard_normal(301).astype(np.float32)
    gs = [rng.standard_normal(301).astype(np.float32) for _ in range(3)]
    # mu = 0: Nesterov and the classical step coincide bit for bit (g + 0*v' = g)
    a, b = orc.Oracle(w0, 3, 1, 0.25, 0.0), orc.Oracle(w0, 3, 1, 0.25, 0.0)
    a.set_nesterov(True)
    for g in gs:
        a.bsp_step([g])
        b.bsp_step([g])
    assert np.array_equal(a.params(), b.params())
    # mu > 0: the first step differs exactly by the look-ahead term eta*mu*v1 (v0 = 0, so v1 = g), fp64
    a, b = (orc.Oracle(w0, 3, 1, 0.25, 0.5, dtype=np.float64) for _ in range(2))
    a.set_nesterov(True)
    a.bsp_step([gs[0]])
    b.bsp_step([gs[0]])
    np.testing.assert_allclose(b.params() - a.params(), 0.25 * 0.5 * gs[0].astype(np.float64), rtol=1e-12,
                               atol=1e-15)
    assert a.set_nesterov(2) != 0


# ---------------------------------------------------------------------------------------------------------------
# BSP == mini-batch SGD on the concatenated batch ("equivalent to a true mini-batch stochastic gradient
# descent algorithm"); n = 1 special case
def _toy(seed=3, N=256, d=33, C=4):
    rng = np.random.default_rng(seed)
    means = rng.standard_normal((C, d - 1)) * 2
    y = rng.integers(0, C, N).astype(np.int32)
    X = np.concatenate([means[y] + rng.standard_normal((N, d - 1)), np.ones((N, 1))], axis=1).astype(np.float32)
    return X, y


def test_bsp_equals_serial_sgd_double(orc):
    X, y = _toy()
    n, B, d, C = 4, 16, X.shape[1], 4
    eta, mu = 0.0625, 0.9                       # power-of-two eta: eta_BSP = n*eta is exact for both runs
    bsp = orc.Oracle(np.zeros(d * C), 2, n, eta, mu, dtype=np.float64)
    ser = orc.Oracle(np.zeros(d * C), 1, 1, n * eta, mu, dtype=np.float64)
    for step in range(200):
        lo = (step * n * B) % X.shape[0]
        idx = np.arange(lo, lo + n * B) % X.shape[0]
        w = bsp.params()
        grads = [orc.softmax_loss_grad(X[idx[j * B:(j + 1) * B]], y[idx[j * B:(j + 1) * B]], w)[1] for j in range(n)]
        assert bsp.bsp_step(grads) == 0
        assert ser.bsp_step([orc.softmax_loss_grad(X[idx], y[idx], ser.params())[1]]) == 0
    assert np.max(np.abs(bsp.params() - ser.params())) < 1e-10


def test_n1_bsp_equals_asp_equals_sgd(orc):
    rng = np.random.default_rng(5)
    w0 = rng.standard_normal(100).astype(np.float32)
    gs = [rng.standard_normal(100).astype(np.float32) for _ in range(5)]
    a = orc.Oracle(w0, 4, 1, 0.1, 0.9)
    b = orc.Oracle(w0, 4, 1, 0.1, 0.9)
    b.switch(ASP, 0)
    for g in gs:
        assert a.bsp_step([g]) == 0
        rc, _, ver = b.pull(0)
        assert b.asp_push(0, g, ver) == (0, 0)
    assert np.array_equal(a.params(), b.params()) and np.array_equal(a.velocity(), b.velocity())


def test_asp_serial_schedule_is_sequential_sgd(orc):
    # pull_j, push_j fully serialised => staleness 0 and parameters == sequential momentum SGD with lr eta_ASP
    X, y = _toy(seed=9)
    n, B, d, C = 4, 8, X.shape[1], 4
    eta, mu = 0.125, 0.9
    o = orc.Oracle(np.zeros(d * C), 2, n, eta, mu, dtype=np.float64)
    o.set_lr_policy(1, 0.0)                     # ASP lr = eta/n = 1/32, exact
    o.switch(ASP, 0)
    ser = orc.Oracle(np.zeros(d * C), 1, 1, eta / n, mu, dtype=np.float64)   # BSP with n = 1 is plain SGD
    for k in range(40):
        j = k % n
        idx = np.arange(k * B, (k + 1) * B) % X.shape[0]
        rc, w, ver = o.pull(j)
        rc, st = o.asp_push(j, orc.softmax_loss_grad(X[idx], y[idx], w)[1], ver)
        assert rc == 0 and st == 0
        ser.bsp_step([orc.softmax_loss_grad(X[idx], y[idx], ser.params())[1]])
    assert np.max(np.abs(o.params() - ser.params())) < 1e-12


# ---------------------------------------------------------------------------------------------------------------
# staleness and the seeded schedule
def test_staleness_all_pull_then_push(orc):
    n = 6
    o = orc.Oracle(np.zeros(10, np.float32), 2, n, 0.1, 0.9)
    o.switch(ASP, 0)
    vers = [o.pull(j, False)[2] for j in range(n)]
    sts = [o.asp_push(j, np.full(10, 0.01, np.float32), vers[j])[1] for j in range(n)]
    assert sts == list(range(n))


def _brute_force_hist(n, per, n_push):
    """Tick-by-tick simulation written independently of the oracle (all periods are multiples of 1000)."""
    base, version, hist, pushes, total, t = [0] * n, 0, collections.Counter(), [0] * n, 0, 0
    nxt = list(per)
    while total < n_push:
        t += 1000
        for j in range(n):
            if total < n_push and nxt[j] == t:
                hist[version - base[j]] += 1
                version += 1
                total += 1
                pushes[j] += 1
                base[j] = version
                nxt[j] = t + per[j]
    return hist, pushes


def _run_schedule(orc, n, kind, worker, P=4):
    o = orc.Oracle(np.zeros(P, np.float32), 1, n, 0.01, 0.0)
    o.switch(ASP, 0)
    base = {}
    sts = []
    g = np.zeros(P, np.float32)
    for k, j in zip(kind, worker):
        if k == 1:
            base[j] = o.pull(int(j), False)[2]
        else:
            rc, st = o.asp_push(int(j), g, base[j])
            assert rc == 0
            sts.append(st)
    return o, sts


def test_straggler_histogram_pin(orc):
    per = [1000] * 7 + [4000]
    kind, worker, tick = orc.schedule(8, per, 60000)
    o, sts = _run_schedule(orc, 8, kind, worker)
    hist = collections.Counter(sts)
    want = {int(a): int(b) for a, b in golden("straggler_hist.txt") if a != "fast_pushes"}
    assert dict(hist) == want
    bf, pushes = _brute_force_hist(8, per, 60000)
    assert dict(bf) == want
    fast = int([b for a, b in golden("straggler_hist.txt") if a == "fast_pushes"][0])
    pw = collections.Counter(int(w) for k, w in zip(kind, worker) if k == 0)
    assert all(pw[j] == fast for j in range(7)) and pw[7] == 2068
    st = o.stats(64)
    assert st["version"] == 60000 and int(st["hist"][28]) == 2068


def test_homogeneous_steady_state(orc):
    n = 5
    kind, worker, tick = orc.schedule(n, [1000] * n, 500)
    _, sts = _run_schedule(orc, n, kind, worker)
    assert sts[:n] == list(range(n)) and set(sts[n:]) == {n - 1}
    assert max(sts) < n                          # S:179's bound holds for equal periods only


def test_schedule_jitter_properties(orc):
    n, J = 4, 100
    kind, worker, tick = orc.schedule(n, [1000] * n, 400, jitter=J, seed=7)
    assert np.all(np.diff(tick) >= 0)            # global order by tick
    pushes = [(t, w) for k, w, t in zip(kind, worker, tick) if k == 0]
    assert pushes == sorted(pushes)              # ties by worker id
    for j in range(n):                           # per-worker gaps T + d, d in [-J, J], d from splitmix64
        ts = [0] + [t for t, w in pushes if w == j]
        for kk in range(1, len(ts)):
            d = (orc.splitmix64(7 ^ (j << 32) ^ kk) % (2 * J + 1)) - J
            assert ts[kk] - ts[kk - 1] == 1000 + d
    # each push is immediately followed by the same worker's pull
    body = list(zip(kind[n:], worker[n:]))
    assert all(body[i][0] == 0 and body[i + 1] == (1, body[i][1]) for i in range(0, len(body), 2))


# ---------------------------------------------------------------------------------------------------------------
# switch semantics
def test_switch_fraction_endpoints(orc):
    rng = np.random.default_rng(11)
    P, n = 300, 4
    w0 = rng.standard_normal(P).astype(np.float32)
    gs = [[rng.standard_normal(P).astype(np.float32) * 0.01 for _ in range(n)] for _ in range(6)]
    # s = 1 (the switch point is never reached within the run) == pure BSP == momentum SGD on the mean of the n
    # gradients at lr n*eta, against a plain numpy fp64 loop
    b = orc.Oracle(w0.astype(np.float64), 3, n, 0.1, 0.9, dtype=np.float64)
    b.switch(ASP, 6)
    lr_bsp = float(np.float32(float(np.float32(0.1)) * n))
    mu = float(np.float32(0.9))
    w, v = w0.astype(np.float64), np.zeros(P)
    for r in range(6):
        assert b.bsp_step([x.astype(np.float64) for x in gs[r]]) == 0
        v = mu * v + np.mean([x.astype(np.float64) for x in gs[r]], axis=0)
        w = w - lr_bsp * v
    assert b.version == 6 and b.stats()["protocol"] == ASP     # the switch takes effect only once version reaches 6
    np.testing.assert_allclose(b.params(), w, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(b.velocity(), v, rtol=1e-13, atol=1e-15)
    # s = 0 == pure ASP from the first update: with every push preceded by its worker's pull (staleness 0), pure
    # ASP is sequential momentum SGD at the ASP lr eta/sqrt(n). Checked against a plain numpy
    # loop in fp64 (the oracle's fp64 instantiation; numpy's separate multiply and add differ from the oracle's FMA
    # by a few fp64 ulps only).
    c = orc.Oracle(w0.astype(np.float64), 3, n, 0.1, 0.9, dtype=np.float64)
    c.switch(ASP, 0)
    # lr and mu cross the C-ABI as fp32 (reading C12): lr = fp32(fp32(0.1)/sqrt(n)), mu = fp32(0.9)
    lr_asp = float(np.float32(float(np.float32(0.1)) / math.sqrt(n)))
    w, v = w0.astype(np.float64), np.zeros(P)
    for r in range(6):
        for j in range(n):
            ver = c.pull(j, False)[2]
            rc, st = c.asp_push(j, gs[r][j].astype(np.float64), ver)
            assert rc == 0 and st == 0
            v = mu * v + gs[r][j].astype(np.float64)
            w = w - lr_asp * v
    assert c.version == 6 * n
    np.testing.assert_allclose(c.velocity(), v, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(c.params(), w, rtol=1e-13, atol=1e-15)


def test_switch_preserves_state_and_drops_inflight(orc):
    rng = np.random.default_rng(12)
    P, n = 64, 2
    o = orc.Oracle(rng.standard_normal(P).astype(np.float32), 2, n, 0.1, 0.9)
    g = rng.standard_normal(P).astype(np.float32)
    o.bsp_step([g, g])
    w, v = o.params(), o.velocity()
    assert o.switch(ASP, 1) == 0 and o.stats()["protocol"] == ASP
    assert np.array_equal(o.params(), w) and np.array_equal(o.velocity(), v) and o.version == 1
    b0 = o.pull(0, False)[2]
    b1 = o.pull(1, False)[2]
    assert o.asp_push(0, g, b0) == (0, 0)
    assert o.switch(BSP, 0) == 0                 # now: worker 1's gradient is in flight
    assert o.asp_push(1, g, b1)[0] == 2          # SS_E_STATE, dropped
    assert o.stats()["dropped"] == 1
    assert o.bsp_step([g, g], versions=[2, 2]) == 0   # every worker implicitly pulled version 2
    assert o.switch(ASP, 10) == 0 and o.switch(BSP, 20) == 2  # one pending switch at a time


def test_version_accounting(orc):
    rng = np.random.default_rng(2)
    o = orc.Oracle(np.zeros(16, np.float32), 2, 2, 0.1, 0.9)
    g = rng.standard_normal(16).astype(np.float32) * 0.01
    vers = []
    for _ in range(3):
        o.bsp_step([g, g])
        vers.append(o.version)
    o.switch(ASP, 0)
    for k in range(5):
        ver = o.pull(k % 2, False)[2]
        o.asp_push(k % 2, g, ver)
        vers.append(o.version)
    assert vers == list(range(1, 9))
    log = o.log()
    assert len(log) == 3 * 2 + 5 and list(log[:, 2]) == [0] * 6 + [0] * 5


# ---------------------------------------------------------------------------------------------------------------
# shard invariance and error paths
def test_shard_invariance(orc):
    rng = np.random.default_rng(4)
    P, n = 1000, 3
    w0 = rng.standard_normal(P).astype(np.float32)
    gs = [[rng.standard_normal(P).astype(np.float32) for _ in range(n)] for _ in range(4)]
    outs = []
    for S in (1, 2, 8, 16):
        o = orc.Oracle(w0, S, n, 0.05, 0.9)
        for r in range(2):
            o.bsp_step(gs[r])
        o.switch(ASP, 0)
        for r in range(2, 4):
            for j in range(n):
                o.asp_push(j, gs[r][j], o.pull(j, False)[2])
        outs.append(o.params())
    assert all(np.array_equal(outs[0], x) for x in outs[1:])


def test_error_paths(orc):
    with pytest.raises(ValueError):
        orc.Oracle(np.zeros(4, np.float32), 1, 0, 0.1, 0.9)
    for bad in [dict(n=257), dict(lr=0.0), dict(mu=1.0), dict(mu=-0.1)]:
        args = dict(n=2, lr=0.1, mu=0.9) | bad
        with pytest.raises(ValueError):
            orc.Oracle(np.zeros(4, np.float32), 1, args["n"], args["lr"], args["mu"])
    o = orc.Oracle(np.zeros(4, np.float32), 1, 2, 0.1, 0.9)
    g = np.ones(4, np.float32)
    assert o.bsp_step([g]) == 3                          # missing worker: SS_E_PROTOCOL
    assert o.bsp_step([g, g], workers=[0, 0]) == 3       # duplicate
    assert o.bsp_step([g, g], versions=[0, 1]) == 4      # SS_E_BARRIER
    assert o.version == 0                                # errors never partially apply
    assert o.asp_push(0, g, 0)[0] == 2                   # ASP push under BSP: SS_E_STATE
    o.switch(ASP, 0)
    assert o.bsp_step([g, g]) == 2
    assert o.asp_push(0, g, 5)[0] == 5                   # version from the future: SS_E_CAUSALITY
    assert o.asp_push(9, g, 0)[0] == 1
    bad = g.copy()
    bad[2] = np.nan
    assert o.asp_push(0, bad, 0)[0] == 6                 # SS_E_DIVERGED, sticky
    assert o.pull(0, False)[0] == 6 and o.switch(BSP, 0) == 6


# ---------------------------------------------------------------------------------------------------------------
# synthetic gradient generator and toy model
def test_splitmix64_reference_vector(orc):
    # Vigna's splitmix64 reference: state 0, first outputs 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4
    assert orc.splitmix64(0) == 0xE220A8397B1DCDAF
    assert orc.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_synth_grad_values(orc):
    g = orc.synth_grad(20241018, 3, 5, 1000, 4096)
    assert g.dtype == np.float32 and np.all(g >= -1 / 128) and np.all(g < 1 / 128)
    q = g.astype(np.float64) * 64 * 2 ** 24 + 2 ** 23          # back to the 24-bit integer h >> 40
    assert np.array_equal(q, np.round(q)) and q.min() >= 0 and q.max() < 2 ** 24
    for t in (0, 1, 4095):
        i = 1000 + t
        h = orc.splitmix64(20241018 ^ ((3 << 56) ^ (5 << 30) ^ i))
        assert q[t] == h >> 40
    assert abs(g.mean()) < 2e-4 and g.std() == pytest.approx(1 / 128 / math.sqrt(3), rel=0.05)


def test_softmax_zero_params_and_fd(orc):
    X, y = _toy(seed=1, N=16, d=9, C=4)
    loss, grad = orc.softmax_loss_grad(X, y, np.zeros(9 * 4))
    assert loss == pytest.approx(math.log(4), rel=1e-15)       # uniform softmax
    rng = np.random.default_rng(0)
    W = rng.standard_normal(9 * 4) * 0.3
    loss, grad = orc.softmax_loss_grad(X, y, W)
    for i in rng.choice(36, 10, replace=False):
        e = np.zeros(36)
        e[i] = 1e-6
        fd = (orc.softmax_loss_grad(X, y, W + e)[0] - orc.softmax_loss_grad(X, y, W - e)[0]) / 2e-6
        assert fd == pytest.approx(grad[i], rel=1e-5, abs=1e-9)
    # gradient rows sum to zero over classes (softmax invariance)
    assert np.allclose(grad.reshape(9, 4).sum(axis=1), 0, atol=1e-12)


# ---------------------------------------------------------------------------------------------------------------
# straggler detector
def test_detector_arithmetic(orc):
    dt = orc.Detector(4, 3)
    thr = [100.0, 100.0, 100.0, 60.0]   # mean 90, sigma_pop = sqrt(300) = 17.32, threshold 72.68
    f1, c1 = dt.window(thr, [1, 1, 1, 1])
    f2, c2 = dt.window(thr, [1, 1, 1, 1])
    assert not f2.any() and not c1 and not c2               # not after 2 windows
    f3, c3 = dt.window(thr, [1, 1, 1, 1])
    assert list(f3) == [False, False, False, True]
    f4, c4 = dt.window([100.0] * 4, [1, 1, 1, 1])           # reset on a clean window
    assert not f4.any()
    dt.window([100.0] * 4, [2, 2, 2, 2])
    assert dt.window([7.0] * 4, [1, 1, 1, 1])[1]            # 3 clean windows: cluster free of stragglers
    dt2 = orc.Detector(4, 1)
    assert not dt2.window([100, 100, 100, 100], [1, 1, 1, 1])[0].any()   # sigma = 0: S_k < S is false
    # two slow of four: mean 80, sigma 20, threshold exactly 60 -> the strict '<' flags nobody
    assert not dt2.window([100, 100, 60, 60], [1, 1, 1, 1])[0].any()
    assert dt2.window([100, 100, 100, 60], [1, 1, 1, 1])[0][3]
    # throughput is samples / busy time: 4x the busy time for the same samples is a 4x slower worker
    assert list(dt2.window([10, 10, 10, 10], [1, 1, 1, 4])[0]) == [False, False, False, True]


def test_detector_masked_arithmetic(orc):
    # Elastic policy (reading C25): only the workers still at the BSP barrier are measured. Hand arithmetic:
    # unmasked (100, 100, 100, 60, 0): S = 72, sigma_pop = sqrt((3*28^2 + 12^2 + 72^2)/5) = sqrt(1536) = 39.19,
    # threshold 32.81 -> only worker 4 is below; with worker 4 masked out the statistics are those of
    # (100, 100, 100, 60): S = 90, sigma = 17.32, threshold 72.68 -> worker 3 is below.
    thr, ones = [100.0, 100.0, 100.0, 60.0, 0.0], [1.0] * 5
    mask = [1, 1, 1, 1, 0]
    assert math.sqrt((3 * 28 ** 2 + 12 ** 2 + 72 ** 2) / 5) == pytest.approx(39.1918, rel=1e-5)
    dt = orc.Detector(5, 3)
    for _ in range(2):                                   # worker 4 below the threshold twice (run = 2, not yet 3)
        f, clean = dt.window(thr, ones)
        assert not f.any() and not clean
    f, _ = dt.window(thr, ones, mask)                    # masked: worker 4 not measured -> its run restarts at 0
    assert not f.any()
    f, _ = dt.window(thr, ones, mask)
    assert not f.any()                                   # worker 3: 2 consecutive windows, not yet K = 3
    f, clean = dt.window(thr, ones, mask)
    assert list(f) == [False, False, False, True, False] and not clean   # worker 3 flagged after 3; worker 4 never
    f, _ = dt.window(thr, ones)                          # unmasked again: worker 4 starts from 1, not 3 (reset),
    assert not f.any()                                   # and worker 3 (60 > 32.81) is no longer below
    f, _ = dt.window(thr, ones)
    assert not f.any()
    f, _ = dt.window(thr, ones)
    assert list(f) == [False, False, False, False, True]
    # a masked-out worker's throughput does not enter S or sigma: masking the slow worker with any value leaves the
    # others' statistics (100, 100, 100, 100) -> sigma = 0, nobody flagged
    dt1 = orc.Detector(5, 1)
    for junk in (0.0, 1e9, 55.0):
        f, _ = dt1.window([100.0] * 4 + [junk], ones, [1, 1, 1, 1, 0])
        assert not f.any()


# ---------------------------------------------------------------------------------------------------------------
# post-switch momentum variants
def _mu_sequence(orc, rule, n=8, mu=0.9, pushes=12, epoch_pushes=2):
    # P = 1; one BSP step with unit gradients makes v = 1; after the switch every push has gradient 1, so
    # v_{k+1} = mu_k * v_k + 1 reveals mu_k = (v_{k+1} - 1) / v_k
    o = orc.Oracle([0.0], 1, n, 0.01, mu, dtype=np.float64)
    assert o.set_momentum_policy(rule, samples_per_epoch=epoch_pushes * 128, batch=128) == 0
    assert o.bsp_step([[1.0]] * n) == 0 and o.velocity()[0] == 1.0
    o.switch(ASP, 0)
    mus = []
    for k in range(pushes):
        v = o.velocity()[0]
        rc, _ = o.asp_push(k % n, [1.0], o.version)
        assert rc == 0
        mus.append((o.velocity()[0] - 1.0) / v)
    return mus


def test_momentum_variants_sequences(orc):
    f32 = lambda x: float(np.float32(x))  # noqa: E731  (mu travels as fp32)
    n, mu = 8, f32(0.9)
    want = {
        0: [mu] * 12,                                                  # same momentum (the paper's choice)
        1: [0.0] * 12,                                                 # (i) 0
        2: [1 / n] * 12,                                               # (ii) 1/n
        3: [1 / 8, 1 / 8, 2 / 8, 2 / 8, 4 / 8, 4 / 8] + [mu] * 6,       # (iii) 2^i/n, capped at the BSP value
        4: [0, 0, 1 / 8, 1 / 8, 2 / 8, 2 / 8, 3 / 8, 3 / 8, 4 / 8, 4 / 8, 5 / 8, 5 / 8],   # (iv) i/n
    }
    for rule, seq in want.items():
        got = _mu_sequence(orc, rule)
        np.testing.assert_allclose(got, seq, rtol=1e-12, atol=1e-15, err_msg=f"rule {rule}")
    # the i/n ramp stops at the BSP momentum too
    assert _mu_sequence(orc, 4, pushes=40)[-1] == pytest.approx(mu, rel=1e-12)


def test_momentum_zero_is_plain_sgd_after_switch(orc):
    rng = np.random.default_rng(21)
    w0 = rng.standard_normal(64).astype(np.float32)
    g = rng.standard_normal(64).astype(np.float32)
    o = orc.Oracle(w0, 2, 1, 0.125, 0.9)
    o.set_momentum_policy(1)
    o.bsp_step([g])                      # builds up v
    o.switch(ASP, 0)
    w1 = o.params()
    assert o.asp_push(0, g, o.version)[0] == 0
    assert np.array_equal(o.velocity(), g)                     # mu = 0: v' = g exactly
    assert np.array_equal(o.params(), (w1.astype(np.float64) - 0.125 * g.astype(np.float64)).astype(np.float32))
