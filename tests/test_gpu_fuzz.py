"""Seeded random protocol programs: the CUDA path (through the C-ABI) against the oracle, call by call.

Each case (tests/fuzz_program.py) draws a shape (P with a ragged tail, S, n), replay window, lr schedule and ASP lr
rule, weight decay, momentum form and (G > 1) exchange mode, then a random program of calls: BSP supersteps
(at one GPU sometimes with a missing worker or a stale base version), ASP pushes from the workers' last pulls
(sometimes from the future, or landing after an ASP->BSP switch and dropped), pulls, and switches at past or future
steps. Every call's status and returned integer (staleness, pull version) must equal the oracle's at once (SV §8b:
integers are returned immediately). Parameters, momentum, every pull snapshot, the staleness log, histogram and
dropped count are compared at the end (and, at one GPU, at random sync points): bit-for-bit at one GPU and in the
exact fused mode (fixed ascending reduction order, reading C12); within C13 after NCCL or pre-summed BSP
supersteps (another summation order). Multi-GPU cases run one torchrun rank per GPU (tests/dist_fuzz_worker.py).
"""
import collections
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from fuzz_program import Program

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 20241018


@pytest.fixture(scope="module")
def ss():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2104_08364_b200 import build
    build.build()
    from paper_2104_08364_b200 import syncswitch
    torch.cuda.init()
    return syncswitch


def run_oracle(orc, prog: Program, on_check=None):
    """The program on the oracle: per-op (status, value) records, snapshots per worker in pull order, final state."""
    P, n = prog.P, prog.n
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    o = orc.Oracle(w0, prog.S, n, 0.1, 0.9)
    o.set_lr_schedule(prog.bounds, prog.factors)
    o.set_lr_policy(prog.asp_rule, prog.lam)
    o.set_nesterov(prog.nesterov)
    k = collections.Counter()
    base, rec, snaps, is_bsp = {}, [], {j: [] for j in range(n)}, []

    def grad(j):
        h = orc.synth_grad(SEED, j, k[j], 0, P)
        k[j] += 1
        return h

    for _ in range(prog.n_ops):
        ver = o.version
        op = prog.next_op(o.stats(1)["protocol"], ver, base)
        is_bsp.append(op[0] == "bsp")
        if op[0] == "bsp":
            js, vers = prog.bsp_call(op, ver, range(n))
            rec.append((o.bsp_step([grad(j) for j in js], js, vers), 0))
        elif op[0] == "push":
            s, st = o.asp_push(op[1], grad(op[1]), op[2])
            rec.append((s, st if s == 0 else 0))
        elif op[0] == "pull":
            s, snap, v = o.pull(op[1])
            base[op[1]] = v
            if op[2]:
                snaps[op[1]].append(snap.copy())
            rec.append((s, v))
        elif op[0] == "switch":
            rec.append((o.switch(op[1], op[2]), 0))
        else:
            if on_check is not None:
                on_check(o)
            rec.append((0, 0))
    return o, np.array(rec, np.int64).reshape(-1, 2), snaps, np.array(is_bsp, bool)


def _single(ss, orc, case_seed):
    prog = Program(case_seed)
    P, n = prog.P, prog.n
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), prog.S, n, 0.1, 0.9)
    g.set_window(prog.window)
    g.set_lr_schedule(prog.bounds, prog.factors)
    g.set_lr_policy(prog.asp_rule, prog.lam)
    g.set_nesterov(prog.nesterov)
    k = collections.Counter()
    keep, base, rec, snaps = [], {}, [], {j: [] for j in range(n)}
    checks = []

    def grad(j):
        d = torch.empty(P, device="cuda")
        assert ss.ss_synth_grad(SEED, j, k[j], 0, P, d) == 0
        k[j] += 1
        keep.append(d)                 # borrowed until the next sync (SV §8b)
        return d

    for _ in range(prog.n_ops):
        ver = g.version
        op = prog.next_op(g.stats(1)["protocol"], ver, base)
        if op[0] == "bsp":
            js, vers = prog.bsp_call(op, ver, range(n))
            rec.append((g.bsp_step_status([grad(j) for j in js], js, vers), 0))
        elif op[0] == "push":
            s, st = g.asp_push_status(op[1], grad(op[1]), op[2])
            rec.append((s, st if s == 0 else 0))
        elif op[0] == "pull":
            dst = torch.empty(P, device="cuda") if op[2] else None
            s, v = ss.ss_pull(g.ctx, op[1], dst)
            base[op[1]] = v
            if dst is not None:
                snaps[op[1]].append(dst)
            rec.append((s, v))
        elif op[0] == "switch":
            rec.append((g.switch_status(op[1], op[2]), 0))
        else:
            g.sync()
            checks.append((g.params(), g.velocity()))
            rec.append((0, 0))
    g.sync()
    o_checks = []
    o, rec_o, snaps_o, _ = run_oracle(orc, Program(case_seed),          # a fresh copy of the same program
                                      on_check=lambda o: o_checks.append((o.params(), o.velocity())))
    assert np.array_equal(np.array(rec, np.int64).reshape(-1, 2), rec_o)
    for (wg, vg), (wo, vo) in zip(checks, o_checks):
        assert np.array_equal(wg, wo) and np.array_equal(vg, vo)
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    for j in range(n):
        assert len(snaps[j]) == len(snaps_o[j])
        for d, h in zip(snaps[j], snaps_o[j]):
            assert np.array_equal(d.cpu().numpy(), h)
    sg, so = g.stats(64), o.stats(64)
    assert (sg["version"], sg["protocol"], sg["dropped"]) == (so["version"], so["protocol"], so["dropped"])
    assert np.array_equal(np.asarray(sg["hist"], np.uint64), np.asarray(so["hist"], np.uint64))
    assert np.array_equal(g.log(), o.log())
    g.close()
    o.close()


@pytest.mark.parametrize("case_seed", list(range(int(os.environ.get("SS_FUZZ_CASES", "64")))))
def test_random_protocol_sequences_bit_exact(ss, orc, case_seed):
    _single(ss, orc, 1000 + case_seed)


def close_c13(x, y, rel=1e-5):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    rms = np.sqrt(np.mean(y * y)) if y.size else 0.0
    return bool(np.all(np.abs(x - y) <= rel * np.abs(y) + rel * rms))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case_seed", list(range(int(os.environ.get("SS_FUZZ_MULTI_CASES", "8")))))
def test_random_protocol_sequences_multi_gpu(orc, world, case_seed):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    seed = 5000 + 100 * world + case_seed
    prog = Program(seed, world)
    with tempfile.TemporaryDirectory() as tmp:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr=127.0.0.1", f"--master-port={29500 + (os.getpid() + case_seed) % 1000}",
               os.path.join(ROOT, "tests", "dist_fuzz_worker.py"), "--out", tmp, "--seed", str(seed)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=180)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        ranks = [dict(np.load(os.path.join(tmp, f"rank{q}.npz"))) for q in range(world)]
    check_multi(orc, prog, ranks)


def check_multi(orc, prog: Program, ranks):
    """Every rank's records (dist_fuzz_worker.py) against the oracle's run of the same program."""
    o, rec_o, snaps_o, is_bsp = run_oracle(orc, prog)
    # bit-exact unless a BSP superstep was applied with another summation order (NCCL or pre-summed mode)
    exact = prog.fused in (1, 3) or not np.any(rec_o[is_bsp, 0] == 0)
    same = np.array_equal if exact else close_c13
    st = o.stats(64)
    for q, d in enumerate(ranks):
        assert np.array_equal(d["rec"], rec_o), f"rank {q}"
        assert int(d["version"]) == st["version"] and int(d["dropped"]) == st["dropped"]
        assert np.array_equal(d["hist"], np.asarray(st["hist"], np.uint64))
        assert np.array_equal(d["log"], o.log())
        assert same(d["w"], o.params()) and same(d["v"], o.velocity()), f"rank {q} (exact={exact})"
        for j in d["hosted"]:
            got = d[f"snaps{int(j)}"]
            assert got.shape[0] == len(snaps_o[int(j)]), f"rank {q} worker {j}"
            for a, b in zip(got, snaps_o[int(j)]):
                assert same(a, b), f"rank {q} worker {j} (exact={exact})"
    o.close()
