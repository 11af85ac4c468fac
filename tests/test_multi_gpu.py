"""Multi-GPU parity (G = 2 and 4 ranks, one process per GPU via torchrun, NCCL over NVLink) against the oracle.

Pure-ASP runs are bit-exact at any G (owner routing moves data, the arithmetic per element is unchanged). Runs with
NCCL BSP supersteps match within the C13 tolerance (NCCL's reduce-scatter summation order differs from ascending
workers) unless the fused peer-memory path (bit-exact, ascending workers) is selected. Protocol
integers are exact in every case. Skipped when the box has fewer GPUs than ranks.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 20241018


def oracle_run(orc, P, n, S, bsp1, pushes, bsp2, drop=-1, bsp_drop=0, idx=None, nesterov=False):
    """The dist_worker call sequence on the oracle; with `idx`, on those elements only (elementwise update: exact for
    them by shard invariance)."""
    if idx is None:
        w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    else:
        w0 = np.array([orc.synth_grad(SEED + 1, 255, 0, int(i), 1)[0] for i in idx], np.float32) * np.float32(64.0)
        S = 1
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    o.set_lr_schedule([bsp1 + 10], [0.5])
    o.set_nesterov(nesterov)
    counter = {j: 0 for j in range(n)}

    def grad(j):
        k = counter[j]
        counter[j] += 1
        if idx is None:
            return orc.synth_grad(SEED, j, k, 0, P)
        return np.array([orc.synth_grad(SEED, j, k, int(i), 1)[0] for i in idx], np.float32)

    for _ in range(bsp1):
        assert o.bsp_step([grad(j) for j in range(n)]) == 0
    if drop >= 0:                                        # elastic: BSP without worker `drop`
        members = [j for j in range(n) if j != drop]
        o.set_members(members)
        for _ in range(bsp_drop):
            assert o.bsp_step([grad(j) for j in members], workers=members) == 0
        o.set_members(list(range(n)))
    o.switch(orc.ASP, 0)
    kind, worker, _ = orc.schedule(n, [1000 + 100 * j for j in range(n)], pushes, jitter=100, seed=7)
    base, stale, snaps = {}, [], {j: [] for j in range(n)}
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            _, s, base[j] = o.pull(j)
            snaps[j].append(s)
        else:
            rc, st = o.asp_push(j, grad(j), base[j])
            assert rc == 0
            stale.append(st)
    o.switch(orc.BSP, 0)
    for _ in range(bsp2):
        assert o.bsp_step([grad(j) for j in range(n)]) == 0
    return o, stale, snaps, kind, worker


def launch(world, args, tmp, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}",
           os.path.join(ROOT, "tests", "dist_worker.py"), "--out", tmp, *map(str, args)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def close_c13(x, y, rel=1e-5):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    rms = np.sqrt(np.mean(y * y))
    return bool(np.all(np.abs(x - y) <= rel * np.abs(y) + rel * rms))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", ["asp_only", "switched", "switched_fused", "switched_presum", "elastic_fused",
                                  "elastic_nccl", "nesterov_fused", "switched_pull", "switched_pull_gbuf",
                                  "elastic_pull"])
def test_multi_gpu_parity(orc, world, case):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S, win = 100003, 8, 8, 7
    bsp1, pushes, bsp2 = (0, 80, 0) if case == "asp_only" else (3, 60, 2)
    fused = {"switched_fused": 1, "switched_presum": 2, "elastic_fused": 1, "nesterov_fused": 1, "switched_pull": 3,
             "switched_pull_gbuf": 3, "elastic_pull": 3}.get(case, 0)
    gbuf = int(case.endswith("gbuf"))       # mode 3 with the gradients written into ss_grad_buffer (zero copy)
    nest = case.startswith("nesterov")
    drop, bsp_drop = (1, 3) if case.startswith("elastic") else (-1, 0)
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", win, "--bsp1", bsp1, "--pushes", pushes,
                       "--bsp2", bsp2, "--fused", fused, "--drop", drop, "--bsp-drop", bsp_drop, "--nesterov", int(nest),
                       "--gbuf", gbuf], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    o, stale, snaps, kind, worker = oracle_run(orc, P, n, S, bsp1, pushes, bsp2, drop, bsp_drop, nesterov=nest)
    exact = fused in (1, 3) or case == "asp_only"   # NCCL / pre-summed: other summation orders (C13)
    ow, ov = o.params(), o.velocity()
    for q, r in enumerate(res):
        # worker placement: the oracle's worker -> GPU map (a1)
        assert [int(j) for j in r["hosted"]] == [j for j in range(n) if orc.worker_host(j, n, world) == q]
        # protocol integers: exact on every rank
        assert list(r["stale"]) == stale
        assert np.array_equal(r["log"], o.log())
        assert int(r["version"]) == o.version and np.array_equal(r["hist"], o.stats(64)["hist"])
        if exact:
            assert np.array_equal(r["w"], ow) and np.array_equal(r["v"], ov)
        else:
            assert close_c13(r["w"], ow) and close_c13(r["v"], ov)
        hosted = [int(j) for j in r["hosted"]]
        want = [s for kd, j in zip(kind, worker) if kd == 1 and int(j) in hosted
                for s in [None]]
        # snapshots of hosted workers in event order
        exp = []
        cnt = {j: 0 for j in hosted}
        for kd, j in zip(kind, worker):
            j = int(j)
            if kd == 1 and j in hosted:
                exp.append(snaps[j][cnt[j]])
                cnt[j] += 1
        assert len(exp) == len(r["snaps"]) == len(want)
        for a, b in zip(r["snaps"], exp):
            assert np.array_equal(a, b) if exact else close_c13(a, b)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fused,nvls", [(1, 0), (2, 0), (3, 0), (1, 1), (2, 1)])
def test_multi_gpu_full_size_sampled(orc, world, fused, nvls):
    """Config 3 at full size (P = 25,557,032, n = S = 8, window 16: the bench's configuration) on `world` GPUs:
    1 BSP superstep, a switch, 16 seeded ASP pushes with pulls, a switch back and 1 BSP superstep; 4,096 sampled
    elements against the oracle (bit-exact in fused-exact mode, C13 in pre-summed mode), integers exact. nvls = 1
    forces the opt-in NVSwitch-multicast broadcast (SS_NVLS=1)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dist_worker import sample_indices
    P, n, S = 25_557_032, 8, 8
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 16, "--bsp1", 1, "--pushes", 16,
                       "--bsp2", 1, "--fused", fused, "--sample", 4096, "--gbuf", int(fused == 3)], tmp,
               env={"SS_NVLS": str(nvls)})
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    if nvls and not all(int(r["nvls"]) for r in res):
        pytest.skip("NVLS multicast unavailable on this box")
    idx = sample_indices(P, 4096)
    o, stale, snaps, kind, worker = oracle_run(orc, P, n, S, 1, 16, 1, idx=idx)
    exact = fused in (1, 3)
    for r in res:
        assert list(r["stale"]) == stale and np.array_equal(r["log"], o.log())
        cmp = np.array_equal if exact else close_c13
        assert cmp(r["w"], o.params()) and cmp(r["v"], o.velocity())
        hosted = [int(j) for j in r["hosted"]]
        exp, cnt = [], {j: 0 for j in hosted}
        for kd, j in zip(kind, worker):
            if kd == 1 and int(j) in hosted:
                exp.append(snaps[int(j)][cnt[int(j)]])
                cnt[int(j)] += 1
        assert len(exp) == len(r["snaps"])
        for a, b in zip(r["snaps"], exp):
            assert cmp(a, b)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape", [(33, 3, 4), (1003, 6, 4), (97, 1, 4), (4099, 5, 8)])
@pytest.mark.parametrize("fused", [0, 1, 2, 3])
def test_multi_gpu_edge_layouts(orc, world, shape, fused):
    """Layouts the bench never uses: ranks hosting no worker (n < G), owner regions past the end of a tiny vector
    (P = 33 on 4 ranks of 32-float shards), one worker for the whole job, n not a multiple of G; every exchange mode.
    Protocol integers exact; parameters bit-exact (fused exact, pure ASP) or within C13 (NCCL / pre-summed BSP)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S = shape
    if S % world:
        pytest.skip("S must be a multiple of the world size")
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 5, "--bsp1", 2, "--pushes", 24,
                       "--bsp2", 2, "--fused", fused], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    o, stale, snaps, kind, worker = oracle_run(orc, P, n, S, 2, 24, 2)
    cmp = np.array_equal if fused in (1, 3) else close_c13
    for r in res:
        assert list(r["stale"]) == stale and np.array_equal(r["log"], o.log())
        assert cmp(r["w"], o.params()) and cmp(r["v"], o.velocity())
        hosted = [int(j) for j in r["hosted"]]
        exp, cnt = [], {j: 0 for j in hosted}
        for kd, j in zip(kind, worker):
            if kd == 1 and int(j) in hosted:
                exp.append(snaps[int(j)][cnt[int(j)]])
                cnt[int(j)] += 1
        assert len(exp) == len(r["snaps"])
        for a, b in zip(r["snaps"], exp):
            assert cmp(a, b)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fused", [1, 2])
@pytest.mark.parametrize("P", [100003, 33])
def test_multi_gpu_nvls_forced(orc, world, fused, P):
    """The opt-in NVSwitch-multicast broadcast forced on at 2 and 4 GPUs (SS_NVLS=1): BSP supersteps
    store each updated slice once through the multicast view. Same results as the P2P broadcast: bit-exact in
    fused-exact mode, C13 in pre-summed mode. Skipped when the driver / fabric offers no multicast."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    n, S = 8, 8
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 7, "--bsp1", 3, "--pushes", 40,
                       "--bsp2", 3, "--fused", fused], tmp, env={"SS_NVLS": "1"})
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    if not all(int(r["nvls"]) for r in res):
        pytest.skip("NVLS multicast unavailable on this box")
    o, stale, snaps, kind, worker = oracle_run(orc, P, n, S, 3, 40, 3)
    cmp = np.array_equal if fused in (1, 3) else close_c13
    for r in res:
        assert list(r["stale"]) == stale and np.array_equal(r["log"], o.log())
        assert cmp(r["w"], o.params()) and cmp(r["v"], o.velocity())
        hosted = [int(j) for j in r["hosted"]]
        exp, cnt = [], {j: 0 for j in hosted}
        for kd, j in zip(kind, worker):
            if kd == 1 and int(j) in hosted:
                exp.append(snaps[int(j)][cnt[int(j)]])
                cnt[int(j)] += 1
        assert len(exp) == len(r["snaps"])
        for a, b in zip(r["snaps"], exp):
            assert cmp(a, b)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fused", [0, 1, 2, 3])
def test_multi_gpu_graph_capture(orc, world, fused):
    """ss_capture_* at G > 1 (SURVEY §8(d) config 2 "with and without CUDA Graphs"): the bench step captured once and
    replayed 6 times on every rank equals 8 ordinary steps of the oracle — the fused kernels' flag epochs come from a
    device counter, so every replay synchronises afresh. Bit-exact in fused-exact mode, C13 otherwise."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S, R = 464_154, 8, 8, 6
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 2 * n, "--fused", fused,
                       "--capture", R], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    o.set_lr_schedule([1 << 40], [0.5])            # dist_worker's capture mode: no boundary in range
    bsp_h = [orc.synth_grad(SEED, j, 0, 0, P) for j in range(n)]
    asp_h = [orc.synth_grad(SEED, j, 1, 0, P) for j in range(n)]
    snaps = {}
    for _ in range(R + 2):
        v = o.version
        assert o.bsp_step(bsp_h, versions=[v] * n) == 0
        o.switch(orc.ASP, 0)
        for j in range(n):
            assert o.asp_push(j, asp_h[j], v + 1) == (0, j)
            snaps[j] = o.pull(j)[1]
        o.switch(orc.BSP, 0)
    cmp = np.array_equal if fused in (1, 3) else close_c13
    for r in res:
        assert int(r["version"]) == o.version == (R + 2) * (1 + n)
        assert np.array_equal(r["log"], o.log()) and np.array_equal(r["hist"], o.stats(64)["hist"])
        assert cmp(r["w"], o.params()) and cmp(r["v"], o.velocity())
        for j, snap in zip(r["hosted"], r["snaps"]):
            assert cmp(snap, snaps[int(j)])


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fused", [1, 2, 3])
def test_multi_gpu_graph_capture_odd_exchanges(orc, world, fused):
    """A captured step holding ONE fused exchange (a BSP superstep): consecutive replays would reuse one inbox buffer,
    so the capture closes with a cross-GPU barrier (ss_capture_end). Eight replays equal ten supersteps of the
    oracle, bit-exact in the exact modes."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S, R = 464_154, 8, 8, 8
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 2 * n, "--fused", fused,
                       "--capture", R, "--capture-bsp-only", 1], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    o.set_lr_schedule([1 << 40], [0.5])
    bsp_h = [orc.synth_grad(SEED, j, 0, 0, P) for j in range(n)]
    for _ in range(R + 2):
        assert o.bsp_step(bsp_h, versions=[o.version] * n) == 0
    cmp = np.array_equal if fused in (1, 3) else close_c13
    for r in res:
        assert int(r["version"]) == o.version == R + 2
        assert np.array_equal(r["log"], o.log()) and np.array_equal(r["hist"], o.stats(64)["hist"])
        assert cmp(r["w"], o.params()) and cmp(r["v"], o.velocity())


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fused", [0, 1, 3])
def test_multi_gpu_host_buffers(orc, world, fused):
    """The e2e path at G > 1: gradients and pull destinations in pinned host memory (staged by the library) —
    same results as device buffers (bit-exact in fused-exact mode)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S = 10007, 8, 8
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 7, "--bsp1", 2, "--pushes", 30,
                       "--bsp2", 1, "--fused", fused, "--host-buffers", 1], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    o, stale, snaps, kind, worker = oracle_run(orc, P, n, S, 2, 30, 1)
    cmp = np.array_equal if fused in (1, 3) else close_c13
    for r in res:
        assert list(r["stale"]) == stale and np.array_equal(r["log"], o.log())
        assert cmp(r["w"], o.params())
        hosted = [int(j) for j in r["hosted"]]
        exp, cnt = [], {j: 0 for j in hosted}
        for kd, j in zip(kind, worker):
            if kd == 1 and int(j) in hosted:
                exp.append(snaps[int(j)][cnt[int(j)]])
                cnt[int(j)] += 1
        for a, b in zip(r["snaps"], exp):
            assert cmp(a, b)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("policy", [0, 1])
def test_multi_gpu_scenario(orc, world, policy):
    """The config-4 scenario runner (greedy / elastic) across `world` GPUs (fused exact): the same switch log and
    results as the oracle's run, bit-exact parameters."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S = 4099, 8, 8
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--window", 16, "--fused", 1, "--bsp1", 0,
                       "--scenario", policy], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    sc = dict(n_workers=n, batch=128, total_samples=600 * 128, quota_num=1, quota_den=2, period=1000, jitter=0,
              sched_seed=7, grad_seed=SEED, slow_worker=n - 1, slow_factor=4, slow_t0=3000, slow_t1=30000,
              window_ticks=4000, K=2, policy=policy)
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    o.set_lr_schedule([10], [0.5])
    log, out = orc.scenario(sc, o, P)
    assert len(log) >= 2                               # the straggler triggered the policy
    for r in res:
        assert [tuple(int(x) for x in e) for e in r["log"]] == log
        assert list(r["res"]) == [out[k] for k in ("bsp_steps", "asp_pushes", "dropped", "end_tick", "version")]
        assert np.array_equal(r["plog"], o.log()) and np.array_equal(r["hist"], o.stats(64)["hist"])
        assert np.array_equal(r["w"], o.params()) and np.array_equal(r["v"], o.velocity())


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fused", [0, 1, 2, 3])
def test_multi_gpu_divergence_reaches_every_rank(orc, world, fused):
    """A non-finite gradient element owned by the last rank: only that rank's kernels see the non-finite update, but
    ss_sync is collective and agrees on the divergence flag, so EVERY rank returns SS_E_DIVERGED at the same ss_sync
    and stays diverged (sticky). The oracle diverges on the same superstep."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    P, n, S = 4099, 8, 8
    with tempfile.TemporaryDirectory() as tmp:
        launch(world, ["--P", P, "--nworkers", n, "--nshards", S, "--bsp1", 2, "--fused", fused, "--nan-bsp", 1], tmp)
        res = [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    for k in range(2):
        assert o.bsp_step([orc.synth_grad(SEED, j, k, 0, P) for j in range(n)]) == 0
    gs = [orc.synth_grad(SEED, j, 2, 0, P) for j in range(n)]
    gs[0][P - 1] = np.nan
    first = o.bsp_step(gs)
    assert first in (0, 6) and o.bsp_step(gs) == 6            # the oracle diverges on this superstep (sticky)
    for r in res:
        s1, s2, s3 = (int(x) for x in r["status"])
        assert s1 in (0, 6) and s2 == 6 and s3 == 6, (s1, s2, s3)
