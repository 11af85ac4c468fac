"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Single GPU: the reduction order is fixed on both sides (ascending workers, explicit FMA; reading C12), so
parameters, momentum and pull snapshots must be BIT-identical, and every protocol integer (version, staleness,
applied order, histogram, dropped count) exact. The toy model's gradient kernel (exp/log in fp32 vs the oracle's
fp64) is compared with the C13 tolerance |x - y| <= 1e-5 |y| + 1e-5 rms(y).
"""
import collections

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 20241018
BSP, ASP = 0, 1


@pytest.fixture(scope="module")
def ss():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2104_08364_b200 import build
    build.build()
    from paper_2104_08364_b200 import syncswitch
    torch.cuda.init()
    return syncswitch


def dev_synth(ss, j, k, P, seed=SEED, offset=0):
    buf = torch.empty(P + offset, dtype=torch.float32, device="cuda")
    out = buf[offset:]
    assert ss.ss_synth_grad(seed, j, k, 0, P, out) == 0
    torch.cuda.synchronize()
    return out


def host_synth(orc, j, k, P, seed=SEED):
    return orc.synth_grad(seed, j, k, 0, P)


def init_params(orc, P):
    return orc.synth_grad(SEED + 1, 255, 0, 0, P) * 64.0   # uniform in [-0.5, 0.5), exact in fp32


def close_c13(x, y, rel=1e-5):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    rms = np.sqrt(np.mean(y * y)) if y.size else 0.0
    return np.all(np.abs(x - y) <= rel * np.abs(y) + rel * rms)


# ---------------------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("j,k,i0,count,offset", [(0, 0, 0, 1, 0), (3, 5, 1000, 4099, 0), (255, 2 ** 26 - 1, 7, 333, 1),
                                                 (7, 12, 2 ** 30 - 4096, 4096, 2)])
def test_synth_grad_bit_exact(ss, orc, j, k, i0, count, offset):
    buf = torch.zeros(count + offset, dtype=torch.float32, device="cuda")
    assert ss.ss_synth_grad(SEED, j, k, i0, count, buf[offset:]) == 0
    got = buf[offset:].cpu().numpy()
    assert np.array_equal(got, orc.synth_grad(SEED, j, k, i0, count))


# ---------------------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("P,n,S", [(1, 1, 1), (7, 2, 3), (1000, 3, 2), (100003, 8, 8), (464154, 8, 8),
                                   (5000, 11, 4), (4096, 16, 16)])
@pytest.mark.parametrize("lam", [0.0, 1e-4])
def test_bsp_bit_exact(ss, orc, P, n, S, lam):
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.05, 0.9)
    o = orc.Oracle(w0, S, n, 0.05, 0.9)
    o64 = orc.Oracle(w0, S, n, 0.05, 0.9, dtype=np.float64)    # the fp64 reference of the same method
    for x in (g, o, o64):
        x.set_lr_schedule([2], [0.1])        # a decay boundary inside the run (version coordinate)
        x.set_lr_policy(0, lam)
    keep = []                                 # gradients are borrowed until ss_sync (SV §8b): supersteps may be deferred
    for step in range(3):
        dg = [dev_synth(ss, j, step, P) for j in range(n)]
        keep += dg
        hg = [host_synth(orc, j, step, P) for j in range(n)]
        perm = list(reversed(range(n)))       # order of submission must not matter (sum is ascending by id)
        g.bsp_step([dg[j] for j in perm], perm, [step] * n)
        assert o.bsp_step(hg) == 0
        assert o64.bsp_step([h.astype(np.float64) for h in hg]) == 0
    assert np.array_equal(g.params(), o.params())          # bit-exact with the same-precision oracle (C12)
    assert np.array_equal(g.velocity(), o.velocity())
    assert close_c13(g.params(), o64.params()) and close_c13(g.velocity(), o64.velocity())   # <= 1e-5 of fp64
    sg, so = g.stats(), o.stats()
    assert sg["version"] == so["version"] == 3 and np.array_equal(sg["hist"], so["hist"])
    assert np.array_equal(g.log(), o.log())
    g.close()


# ---------------------------------------------------------------------------------------------------------------
def run_asp_pair(ss, orc, P, n, S, kind, worker, window, host_buffers=False, offset=0, lam=0.0):
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    o64 = orc.Oracle(w0, S, n, 0.1, 0.9, dtype=np.float64)
    for x in (g, o, o64):
        x.set_lr_schedule([60], [0.5])
        x.set_lr_policy(0, lam)
        x.switch(ASP, 0)
    g.set_window(window)
    base_g, base_o = {}, {}
    pulls_g, pulls_o, st_g, st_o = [], [], [], []
    keep = []
    pushes = collections.Counter()
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            if host_buffers:
                dst = np.empty(P, np.float32)
            else:
                dst = torch.empty(P + offset, dtype=torch.float32, device="cuda")[offset:]
            base_g[j] = g.pull(j, dst)
            rc, snap, base_o[j] = o.pull(j)
            pulls_g.append(dst)
            pulls_o.append(snap)
        else:
            k = pushes[j]
            pushes[j] += 1
            if host_buffers:
                grad = host_synth(orc, j, k, P)
            else:
                grad = dev_synth(ss, j, k, P, offset=offset)
            keep.append(grad)                  # borrowed until sync
            st_g.append(g.asp_push(j, grad, base_g[j]))
            rc, s = o.asp_push(j, host_synth(orc, j, k, P), base_o[j])
            assert rc == 0
            st_o.append(s)
            assert o64.asp_push(j, host_synth(orc, j, k, P).astype(np.float64), base_o[j])[0] == 0
    g.sync()
    assert close_c13(g.params(), o64.params())           # within the north-star tolerance of the fp64 result
    return g, o, pulls_g, pulls_o, st_g, st_o


@pytest.mark.parametrize("window", [1, 7, 16, 64])
@pytest.mark.parametrize("P,S", [(10007, 4), (4096, 1)])
def test_asp_bit_exact(ss, orc, window, P, S):
    n = 4
    kind, worker, tick = orc.schedule(n, [1000, 1100, 1300, 1700], 120, jitter=100, seed=7)
    g, o, pg, po, sg, so = run_asp_pair(ss, orc, P, n, S, kind, worker, window)
    assert sg == so and max(so) > 0
    for a, b in zip(pg, po):
        assert np.array_equal(a.cpu().numpy(), b)          # every snapshot sees exactly the pushes before it
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert np.array_equal(g.log(), o.log())
    assert np.array_equal(g.stats()["hist"], o.stats()["hist"])
    g.close()


@pytest.mark.parametrize("window", [2, 16])
def test_asp_host_buffers_and_weight_decay(ss, orc, window):
    # host gradients and pull destinations: staged on the copy streams (H2D / D2H overlapping the kernels)
    n, P = 3, 3001
    kind, worker, _ = orc.schedule(n, [1000] * n, 40, jitter=100, seed=3)
    g, o, pg, po, sg, so = run_asp_pair(ss, orc, P, n, 2, kind, worker, window, host_buffers=True, lam=1e-3)
    assert sg == so
    for a, b in zip(pg, po):
        assert np.array_equal(a, b)
    assert np.array_equal(g.params(), o.params())
    g.close()


def test_asp_unaligned_scalar_path(ss, orc):
    n, P = 2, 2053
    kind, worker, _ = orc.schedule(n, [1000, 1500], 30, jitter=0)
    g, o, pg, po, sg, so = run_asp_pair(ss, orc, P, n, 1, kind, worker, 8, offset=1)
    for a, b in zip(pg, po):
        assert np.array_equal(a.cpu().numpy(), b)
    assert np.array_equal(g.params(), o.params())
    g.close()


def test_straggler_histogram_on_gpu(ss, orc):
    # config 4 shape (SURVEY §8c pin): the staleness integers through the C-ABI match the brute-force pin
    n, P = 8, 64
    kind, worker, _ = orc.schedule(n, [1000] * 7 + [4000], 3000)
    g, o, pg, po, sg, so = run_asp_pair(ss, orc, P, n, 8, kind, worker, 64)
    assert sg == so
    assert collections.Counter(sg)[28] == collections.Counter(so)[28] > 0
    assert np.array_equal(g.params(), o.params())
    g.close()


# ---------------------------------------------------------------------------------------------------------------
def test_switch_bsp_asp_bsp_bit_exact(ss, orc):
    n, S, P = 4, 4, 9999
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    for x in (g, o):
        x.set_lr_schedule([5, 9], [0.1, 0.01])
    k = collections.Counter()

    def grads(js):
        out_d, out_h = [], []
        for j in js:
            out_d.append(dev_synth(ss, j, k[j], P))
            out_h.append(host_synth(orc, j, k[j], P))
            k[j] += 1
        return out_d, out_h

    keep = []
    for step in range(3):
        d, h = grads(range(n))
        keep += d
        g.bsp_step(d)
        assert o.bsp_step(h) == 0
    assert g.switch_status(ASP, 3) == o.switch(ASP, 3) == 0
    assert g.stats()["protocol"] == o.stats()["protocol"] == ASP
    dst_g = {j: torch.empty(P, device="cuda") for j in range(n)}
    bg = {j: g.pull(j, dst_g[j]) for j in range(n)}
    bo = {j: o.pull(j)[2] for j in range(n)}
    for j in (2, 0, 3):                               # three pushes land, worker 1's stays in flight
        d, h = grads([j])
        keep += d
        assert g.asp_push(j, d[0], bg[j]) == o.asp_push(j, h[0], bo[j])[1]
    assert g.switch_status(BSP, 0) == o.switch(BSP, 0) == 0
    d, h = grads([1])
    assert g.asp_push_status(1, d[0], bg[1])[0] == o.asp_push(1, h[0], bo[1])[0] == 2   # dropped
    assert g.stats()["dropped"] == o.stats()["dropped"] == 1
    assert g.version == o.version == 6
    for step in range(4):                             # across the decay boundaries at 9
        d, h = grads(range(n))
        keep += d
        g.bsp_step(d, versions=[6 + step] * n)
        assert o.bsp_step(h, versions=[6 + step] * n) == 0
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert np.array_equal(g.log(), o.log())
    g.close()


def test_switch_fraction_endpoints_on_gpu(ss, orc):
    # s = 1 (switch beyond the run) == pure BSP;  s = 0 == pure ASP — on the device path
    n, S, P = 2, 2, 4099
    w0 = init_params(orc, P)
    a = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    b = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    b.switch(ASP, 4)
    keep = []
    for step in range(4):
        gs = [dev_synth(ss, j, step, P) for j in range(n)]
        keep += gs
        a.bsp_step(gs)
        b.bsp_step(gs)
    assert np.array_equal(a.params(), b.params())
    assert b.stats()["protocol"] == ASP
    a.close()
    b.close()


# ---------------------------------------------------------------------------------------------------------------
def test_errors_match_oracle(ss, orc):
    P, n = 64, 2
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), 1, n, 0.1, 0.9)
    o = orc.Oracle(w0, 1, n, 0.1, 0.9)
    x = dev_synth(ss, 0, 0, P)
    h = host_synth(orc, 0, 0, P)
    assert g.bsp_step_status([x]) == o.bsp_step([h]) == ss.SS_E_PROTOCOL
    assert g.bsp_step_status([x, x], [1, 1]) == o.bsp_step([h, h], workers=[1, 1]) == ss.SS_E_PROTOCOL
    assert g.bsp_step_status([x, x], [0, 1], [0, 1]) == o.bsp_step([h, h], versions=[0, 1]) == ss.SS_E_BARRIER
    assert g.asp_push_status(0, x, 0)[0] == o.asp_push(0, h, 0)[0] == ss.SS_E_STATE
    assert g.version == o.version == 0
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    assert g.bsp_step_status([x, x]) == o.bsp_step([h, h]) == ss.SS_E_STATE
    assert g.asp_push_status(0, x, 3)[0] == o.asp_push(0, h, 3)[0] == ss.SS_E_CAUSALITY
    assert g.asp_push_status(5, x, 0)[0] == o.asp_push(5, h, 0)[0] == ss.SS_E_INVAL
    assert g.switch_status(BSP, 10) == o.switch(BSP, 10) == 0
    assert g.switch_status(ASP, 20) == o.switch(ASP, 20) == ss.SS_E_STATE
    assert g.stats()["dropped"] == o.stats()["dropped"] == 1
    g.close()


def test_divergence_is_sticky(ss, orc):
    P = 1000
    g = ss.SyncSwitch(torch.zeros(P, device="cuda"), 2, 1, 0.1, 0.9)
    bad = torch.zeros(P, device="cuda")
    bad[17] = float("nan")
    g.bsp_step([bad])
    assert g.sync_status() == ss.SS_E_DIVERGED
    assert g.bsp_step_status([bad]) == ss.SS_E_DIVERGED
    assert g.switch_status(ASP, 0) == ss.SS_E_DIVERGED
    g.close()
    g = ss.SyncSwitch(torch.zeros(P, device="cuda"), 2, 1, 0.1, 0.9)
    g.switch(ASP, 0)
    inf = torch.zeros(P, device="cuda")
    inf[999] = float("inf")
    g.asp_push(0, inf, 0)
    assert g.sync_status() == ss.SS_E_DIVERGED
    g.close()


def test_repeated_init_destroy(ss):
    for _ in range(20):
        g = ss.SyncSwitch(torch.zeros(1 << 16, device="cuda"), 4, 4, 0.1, 0.9)
        g.close()


@pytest.mark.parametrize("window", [2, 16])
def test_host_buffers_full_size_slot_reuse(ss, orc, window):
    """The e2e pattern at config 3 size: pinned host gradients and a distinct pinned host destination for every pull,
    three ASP rounds (each push followed by its pull). Staging slots are reused across windows while earlier D2H
    copies may still be running (window 2: every window reuses the ring); every snapshot must equal the oracle's on
    4,096 sampled elements."""
    P, n, S = 25_557_032, 8, 8
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([rng.choice(P, 4090, replace=False), [0, 1, P - 2, P - 1]]))
    ti = torch.from_numpy(idx).cuda()
    w0d = torch.empty(P, device="cuda")
    ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0d)
    g = ss.SyncSwitch(w0d, S, n, 0.1, 0.9)
    g.set_window(window)
    o = orc.Oracle(w0d[ti].cpu().numpy(), 1, n, 0.1, 0.9)
    del w0d
    hgrad, sgrad = {}, {}
    for j in range(n):
        for r in range(2):
            d = dev_synth(ss, j, r, P)
            hgrad[(j, r)] = torch.empty(P, pin_memory=True)
            hgrad[(j, r)].copy_(d)
            sgrad[(j, r)] = d[ti].cpu().numpy()
            del d
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    base_g = {j: g.pull(j) for j in range(n)}
    base_o = {j: o.pull(j, False)[2] for j in range(n)}
    snaps, expected = [], []
    for rnd in range(3):
        for j in range(n):
            assert g.asp_push(j, hgrad[(j, rnd % 2)], base_g[j]) == o.asp_push(j, sgrad[(j, rnd % 2)], base_o[j])[1]
            dst = torch.empty(P, pin_memory=True)
            base_g[j] = g.pull(j, dst)
            rc, snap, base_o[j] = o.pull(j)
            snaps.append(dst)
            expected.append(snap)
    g.sync()
    hidx = torch.from_numpy(idx)
    for got, want in zip(snaps, expected):
        assert np.array_equal(got[hidx].numpy(), want)
    assert np.array_equal(g.params()[idx], o.params())
    g.close()


# ---------------------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("P", [25_557_032, 100_000_000, 1_000_000_000])
def test_full_size_sampled(ss, orc, P):
    """BASELINE configs 3 and 5 at full size (P = 25,557,032; 1e8; 1e9 with n = S = 8) in the bench's launch
    configuration (window 16): the oracle is checked on 4,096 sampled elements — the update is elementwise, so an
    oracle built on those indices only (shard invariance) is exact for them."""
    n, S = 8, 8
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.choice(P, 4090, replace=False), [0, 1, P - 2, P - 1]]))
    w0d = torch.empty(P, device="cuda")
    ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0d)
    w0d *= 64.0
    g = ss.SyncSwitch(w0d, S, n, 0.1, 0.9)
    del w0d
    g.set_window(16)
    w0s = np.array([orc.synth_grad(SEED + 1, 255, 0, int(i), 1)[0] * 64.0 for i in idx], np.float32)
    o = orc.Oracle(w0s, 1, n, 0.1, 0.9)

    def sample(j, k):
        return np.array([orc.synth_grad(SEED, j, k, int(i), 1)[0] for i in idx], np.float32)

    grads = [dev_synth(ss, j, 0, P) for j in range(n)]
    g.bsp_step(grads)
    o.bsp_step([sample(j, 0) for j in range(n)])
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    snaps = [torch.empty(P, device="cuda") for _ in range(n)]
    for j in range(n):
        g.pull(j, snaps[j])
        o.pull(j, False)
    g.sync()
    expected = []
    for j in range(n):                               # one round: 8 pushes, each followed by its pull
        ss.ss_synth_grad(SEED, j, 1, 0, P, grads[j])  # ring slot 1 (the BSP step's reads completed at the sync)
        assert g.asp_push(j, grads[j], 1) == j
        assert o.asp_push(j, sample(j, 1), 1) == (0, j)
        g.pull(j, snaps[j])
        expected.append(o.pull(j)[1])
    g.sync()
    ti = torch.from_numpy(idx).cuda()
    want = o.params()
    for j in range(n):                               # pull j sees exactly the first j + 1 pushes
        assert np.array_equal(snaps[j][ti].cpu().numpy(), expected[j])
    assert np.array_equal(expected[n - 1], want)
    if P <= 100_000_000:                                             # full host copies of w, v stay small
        assert np.array_equal(g.params()[idx], want)
        assert np.array_equal(g.velocity()[idx], o.velocity())
    g.close()


# ---------------------------------------------------------------------------------------------------------------
def test_softmax_grad_kernel(ss, orc):
    from inputs import toy_dataset
    X, y = toy_dataset(seed=1, n_points=64)
    B, d, C = 16, X.shape[1], 8
    rng = np.random.default_rng(0)
    W = (rng.standard_normal(d * C) * 0.01).astype(np.float32)
    Xd, yd, Wd = torch.from_numpy(X[:B]).cuda(), torch.from_numpy(y[:B]).cuda(), torch.from_numpy(W).cuda()
    grad = torch.empty(d * C, device="cuda")
    loss = torch.empty(1, device="cuda")
    assert ss.ss_softmax_grad(Xd, yd, B, d, C, Wd, grad, loss) == 0
    lo, go = orc.softmax_loss_grad(X[:B], y[:B], W.astype(np.float64))
    # elementwise within the a-priori fp32 bound of the kernel's operation order (tests/criterion_bounds.py)
    from criterion_bounds import softmax_grad_bounds
    Eg = softmax_grad_bounds(X[:B], y[:B], W.astype(np.float64))["Eg"]
    assert np.all(np.abs(grad.cpu().numpy() - go) <= Eg + 1e-12 * np.abs(go))
    assert close_c13(grad.cpu().numpy(), go) and abs(loss.item() - lo) <= 1e-5 * abs(lo)
    # zero parameters: loss = ln C exactly up to fp32 rounding
    assert ss.ss_softmax_grad(Xd, yd, B, d, C, torch.zeros(d * C, device="cuda"), grad, loss) == 0
    assert loss.item() == pytest.approx(np.log(C), rel=1e-6)


def test_config1_toy_end_to_end(ss, orc):
    """Config 1: 2 workers, 2 shards, softmax regression on 1,000 points (P = 8,192), W = 100 B samples, switch
    BSP -> ASP at s = 0.5 (25 BSP steps + 50 ASP pushes, Table I arithmetic), seeded jittered schedule, overlapping
    classes (inputs.TOY_RECIPE) so the loss is still falling at the switch (start with BSP, switch once).
    Each side computes its own gradients from its own pulls (GPU: softmax_grad kernel fp32; oracle: fp64).
    Checked: protocol integers exact; parameters and the two per-update loss curves within C13; the loss falls
    across the BSP phase AND across the ASP phase; held-out accuracy agrees."""
    from inputs import minibatch_order, toy_split
    n, S, B, d, C = 2, 2, 16, 1024, 8
    X, y, Xte, yte = toy_split()
    bsp_steps, asp_pushes, _ = orc.table1(100 * B, B, n, 1, 2, [])
    assert (bsp_steps, asp_pushes) == (25, 50)
    order = minibatch_order(1, len(X), n * bsp_steps + asp_pushes, B)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    P = d * C
    g = ss.SyncSwitch(torch.zeros(P, device="cuda"), S, n, 0.1, 0.9)
    o = orc.Oracle(np.zeros(P, np.float32), S, n, 0.1, 0.9)
    for x in (g, o):
        x.switch(ASP, bsp_steps)
    loss = torch.empty(1, device="cuda")
    mb = iter(range(len(order)))
    losses_g, losses_o = [], []

    def gpu_grad(Wdev, batch):
        bi = torch.from_numpy(order[batch]).cuda()
        gr = torch.empty(P, device="cuda")
        assert ss.ss_softmax_grad(Xd[bi].contiguous(), yd[bi].contiguous(), B, d, C, Wdev, gr, loss) == 0
        losses_g.append(loss.item())
        return gr

    def orc_grad(Wh, batch):
        lo, go = orc.softmax_loss_grad(X[order[batch]], y[order[batch]], Wh.astype(np.float64))
        losses_o.append(lo)
        return go.astype(np.float32)

    wdev = torch.empty(P, device="cuda")
    for step in range(bsp_steps):
        batches = [next(mb) for _ in range(n)]
        g.pull(0, wdev)
        g.sync()
        g.bsp_step([gpu_grad(wdev, b) for b in batches])
        wo = o.params()
        assert o.bsp_step([orc_grad(wo, b) for b in batches]) == 0
    kind, worker, _ = orc.schedule(n, [1000] * n, asp_pushes, jitter=100, seed=7)
    snap_g = {j: torch.empty(P, device="cuda") for j in range(n)}
    snap_o, base_g, base_o = {}, {}, {}
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            base_g[j] = g.pull(j, snap_g[j])
            _, snap_o[j], base_o[j] = o.pull(j)
            g.sync()
        else:
            b = next(mb)
            sg = g.asp_push(j, gpu_grad(snap_g[j], b), base_g[j])
            g.sync()
            rc, so = o.asp_push(j, orc_grad(snap_o[j], b), base_o[j])
            assert rc == 0 and sg == so
    assert g.version == o.version == bsp_steps + asp_pushes
    assert np.array_equal(g.log(), o.log())
    wg, wo = g.params(), o.params()
    assert close_c13(wg, wo)
    assert close_c13(losses_g, losses_o)
    lo = np.array(losses_o)
    k = n * bsp_steps
    # still training at the switch, and the ASP phase keeps reducing the loss
    assert lo[k - 10:k].mean() < lo[:10].mean() - 0.05 and lo[-10:].mean() < lo[k - 10:k].mean() - 0.05
    acc_g = float(np.mean(np.argmax(Xte @ wg.reshape(d, C), 1) == yte))
    acc_o = float(np.mean(np.argmax(Xte @ wo.reshape(d, C), 1) == yte))
    assert abs(acc_g - acc_o) <= 0.005 and acc_o > 0.5
    g.close()


@pytest.mark.parametrize("P,off", [(5003, 0), (4099, 1)])
def test_nesterov_bit_exact(ss, orc, P, off):
    """Nesterov momentum (reading C28) through bsp_update and the replay kernels (TMA form for 16-byte-aligned
    buffers, the scalar form for misaligned ones; ragged P), bit-exact with the fp32 oracle."""
    n, S = 4, 3
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    g.set_nesterov(True)
    assert o.set_nesterov(True) == 0
    keep = []

    def dev(j, k):
        buf = torch.empty(P + off, device="cuda")
        ss.ss_check(ss.ss_synth_grad(SEED, j, k, 0, P, buf[off:]))
        keep.append(buf)
        return buf[off:]

    for step in range(3):
        g.bsp_step([dev(j, step) for j in range(n)])
        assert o.bsp_step([host_synth(orc, j, step, P) for j in range(n)]) == 0
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    g.set_window(6)
    kind, worker, _ = orc.schedule(n, [1000, 1100, 1300, 1600], 24, jitter=100, seed=9)
    base_g, base_o, cnt = {}, {}, collections.Counter()
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            base_g[j] = g.pull(j)
            base_o[j] = o.pull(j, False)[2]
        else:
            k = 3 + cnt[j]
            cnt[j] += 1
            assert g.asp_push(j, dev(j, k), base_g[j]) == o.asp_push(j, host_synth(orc, j, k, P), base_o[j])[1]
    g.switch(BSP, 0)
    o.switch(BSP, 0)
    g.bsp_step([dev(j, 100) for j in range(n)])
    assert o.bsp_step([host_synth(orc, j, 100, P) for j in range(n)]) == 0
    g.sync()
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert np.array_equal(g.log(), o.log())
    g.close()


@pytest.mark.parametrize("rule", [1, 2, 3, 4])
def test_momentum_policies_bit_exact(ss, orc, rule):
    """Post-switch momentum variants: per-push momentum in the replay kernel, bit-exact with the oracle."""
    n, S, P = 4, 2, 5003
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    for x in (g, o):
        x.set_momentum_policy(rule, samples_per_epoch=3 * 64, batch=64)
    keep = []
    for step in range(2):
        d = [dev_synth(ss, j, step, P) for j in range(n)]
        keep += d
        g.bsp_step(d)
        assert o.bsp_step([host_synth(orc, j, step, P) for j in range(n)]) == 0
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    g.set_window(5)
    kind, worker, _ = orc.schedule(n, [1000, 1200, 1500, 1700], 30, jitter=100, seed=5)
    base_g, base_o, cnt = {}, {}, collections.Counter()
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            base_g[j] = g.pull(j)
            base_o[j] = o.pull(j, False)[2]
        else:
            k = 2 + cnt[j]
            cnt[j] += 1
            d = dev_synth(ss, j, k, P)
            keep.append(d)
            assert g.asp_push(j, d, base_g[j]) == o.asp_push(j, host_synth(orc, j, k, P), base_o[j])[1]
    g.sync()
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    g.close()


def test_graph_capture_replay_bit_exact(ss, orc):
    """ss_capture_* (CUDA graph of one BSP + switch + ASP round + switch step, replayed K times) gives exactly the
    protocol state and parameters of K + 1 ordinary steps (oracle)."""
    n, S, P = 4, 4, 464154
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    g.set_window(2 * n)
    bsp_g = [dev_synth(ss, j, 0, P) for j in range(n)]
    asp_g = [dev_synth(ss, j, 1, P) for j in range(n)]
    dst = [torch.empty(P, device="cuda") for _ in range(n)]
    bsp_h = [host_synth(orc, j, 0, P) for j in range(n)]
    asp_h = [host_synth(orc, j, 1, P) for j in range(n)]

    def gpu_step():
        v = g.version
        g.bsp_step(bsp_g, list(range(n)), [v] * n)
        g.switch(ASP, 0)
        for j in range(n):
            assert g.asp_push(j, asp_g[j], v + 1) == j
            g.pull(j, dst[j])
        g.switch(BSP, 0)

    def orc_step():
        v = o.version
        assert o.bsp_step(bsp_h, versions=[v] * n) == 0
        o.switch(ASP, 0)
        for j in range(n):
            assert o.asp_push(j, asp_h[j], v + 1) == (0, j)
            o.pull(j, False)
        o.switch(BSP, 0)

    gpu_step()                      # warm-up (first use allocates nothing afterwards)
    orc_step()
    g.capture_begin()
    gpu_step()
    assert g.capture_end() == 1 + n
    orc_step()
    g.capture_replay(5)
    for _ in range(5):
        orc_step()
    g.sync()
    assert g.version == o.version == 7 * (1 + n)
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert np.array_equal(g.log(), o.log()) and np.array_equal(g.stats()["hist"], o.stats()["hist"])
    assert np.array_equal(dst[n - 1].cpu().numpy(), o.params())
    g.set_lr_schedule([100], [0.5])                 # a boundary inside the replay range is refused
    with pytest.raises(ss.SSError):
        g.capture_replay(20)
    g.close()


def test_bsp_host_gradients_reuse_slots(ss, orc):
    """BSP supersteps from host gradients, twice per slot set, then an ASP round with host pulls: the copy streams
    must respect slot reuse (a refill waits for the previous consumer)."""
    n, S, P = 4, 2, 70001
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    for step in range(4):
        hg = [host_synth(orc, j, step, P) for j in range(n)]
        g.bsp_step(hg)                                   # no sync between steps: staging slots are reused
        assert o.bsp_step(hg) == 0
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    g.set_window(2)
    outs = [np.empty(P, np.float32) for _ in range(n)]
    for j in range(n):
        hg = host_synth(orc, j, 9, P)
        g.asp_push(j, hg, 4)
        o.asp_push(j, hg, 4)
        g.pull(j, outs[j])
    g.sync()
    assert np.array_equal(g.params(), o.params())
    assert np.array_equal(outs[n - 1], o.params())
    g.close()


def test_max_workers_bsp(ss, orc):
    """The maximum cluster the C-ABI accepts (n = 256 workers in one superstep, S = 64 shards)."""
    n, S, P = 256, 64, 20011
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.001, 0.9)
    o = orc.Oracle(w0, S, n, 0.001, 0.9)
    keep = []
    for step in range(2):
        dg = [dev_synth(ss, j, step, P) for j in range(n)]
        keep += dg                                     # borrowed until ss_sync (SV §8b)
        g.bsp_step(dg)
        assert o.bsp_step([host_synth(orc, j, step, P) for j in range(n)]) == 0
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert g.stats(2)["hist"][0] == 2 * n
    g.close()


# ---------------------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("mode", ["device", "unaligned", "host", "flushed"])
@pytest.mark.parametrize("P,n,S,window", [(100003, 8, 8, 16), (4099, 3, 2, 5), (2 ** 20 + 3, 8, 8, 64)])
def test_windows_with_bsp_supersteps(ss, orc, mode, P, n, S, window):
    """One GPU: BSP supersteps join the pending window (one kernel applies supersteps, pushes and pulls tile by tile,
    w and v on chip). A long program without sync points — 20 supersteps (crossing the window's 128-gradient cap at
    n = 8), a switch, a seeded ASP phase with pulls, a switch back, more supersteps, an lr boundary inside — is
    bit-identical to the oracle for device, unaligned (scalar kernel) and host (staged) gradients, and with ss_flush
    after every call (every superstep and push its own kernel: the bench's form)."""
    w0 = init_params(orc, P)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    g.set_window(window)
    for x in (g, o):
        x.set_lr_schedule([17, 40], [0.5, 0.25])
    k = {j: 0 for j in range(n)}
    keep = []

    def grad(j):
        kk = k[j]
        k[j] += 1
        h = host_synth(orc, j, kk, P)
        if mode == "host":
            d = torch.from_numpy(h).pin_memory() if kk % 2 else h          # pinned and pageable
        else:
            d = dev_synth(ss, j, kk, P, offset=1 if mode == "unaligned" else 0)
        keep.append(d)
        return d, h

    def bsp_round():
        gs = [grad(j) for j in range(n)]
        v = o.version
        g.bsp_step([x[0] for x in gs], list(range(n)), [v] * n)
        if mode == "flushed":
            g.flush()                     # ss_flush: issue the device work now (the bench's dependency points)
        assert o.bsp_step([x[1] for x in gs]) == 0

    for _ in range(20):
        bsp_round()
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    kind, worker, _ = orc.schedule(n, [1000 + 50 * j for j in range(n)], 30, jitter=100, seed=7)
    base_g, base_o, snaps = {}, {}, []
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            dst = torch.empty(P, device="cuda") if mode != "host" else np.zeros(P, np.float32)
            base_g[j] = g.pull(j, dst)
            _, s_o, base_o[j] = o.pull(j)
            snaps.append((dst, s_o))
        else:
            d, h = grad(j)
            sg = g.asp_push(j, d, base_g[j])
            if mode == "flushed":
                g.flush()
            rc, so = o.asp_push(j, h, base_o[j])
            assert rc == 0 and sg == so
    g.switch(BSP, 0)
    o.switch(BSP, 0)
    for _ in range(5):
        bsp_round()
    g.sync()
    assert g.version == o.version == 25 + 30
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert np.array_equal(g.log(), o.log()) and np.array_equal(g.stats()["hist"], o.stats()["hist"])
    for d, s_o in snaps:
        got = d.cpu().numpy() if hasattr(d, "cpu") else d
        assert np.array_equal(got, s_o)
    g.close()
