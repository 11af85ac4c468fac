"""CPU checks of the C-ABI library: it loads without a GPU, exports every symbol include/syncswitch.h declares, and its
host-only control plane (Table I, arrival schedule, detector, greedy policy) agrees bit-exactly with the oracle.
No compute calls are made here (no GPU)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


@pytest.fixture(scope="module")
def ss():
    from paper_2104_08364_b200 import build
    build.build()
    from paper_2104_08364_b200 import syncswitch
    return syncswitch


def _declared():
    src = open(os.path.join(ROOT, "include", "syncswitch.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(ss):
    import subprocess
    declared = _declared()
    assert len(declared) >= 30
    out = subprocess.check_output(["nm", "-D", "--defined-only", ss.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [d for d in declared if d not in exported]
    assert not missing, missing
    assert sorted(ss.EXPORTS) == declared       # the binding wraps exactly the declared surface


def test_library_is_sm100a(ss):
    import subprocess
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ss.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_no_oracle_on_product_path():
    # the product package never imports / links / names the oracle
    pkg = os.path.join(ROOT, "paper_2104_08364_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|oracle\.h|\borc[fd]?_\w+\s*\()",
                                     text), f


def test_init_without_gpu_fails_loudly(ss):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    s, ctx = ss.ss_init(np.zeros(8, np.float32), 8, 1, 1, 0.1, 0.9)
    assert s == ss.SS_E_CUDA and ctx is None
    # argument validation happens before any device work
    for args in [(0, 1, 1, 0.1, 0.9), (8, 0, 1, 0.1, 0.9), (8, 1, 257, 0.1, 0.9), (8, 1, 1, 0.0, 0.9),
                 (8, 1, 1, 0.1, 1.0)]:
        assert ss.ss_init(np.zeros(8, np.float32), *args)[0] == ss.SS_E_INVAL


def test_table1_matches_paper_and_oracle(ss, orc):
    W, B, N = 64000 * 128, 128, 8
    for row in golden("table1.txt"):
        sb, sa, bsp, asp, total, b1, b2 = map(int, row)
        s, got = ss.ss_table1(W, B, N, sb, 100, [32000 * 128, 48000 * 128])
        assert s == 0 and got == (bsp, asp, [b1, b2])
        assert got == orc.table1(W, B, N, sb, 100, [32000 * 128, 48000 * 128])
    assert ss.ss_table1(W, B, N, 1, 3, [])[0] == ss.SS_E_INVAL      # non-integral share


@pytest.mark.parametrize("case", [
    dict(n=8, period=[1000] * 7 + [4000], n_push=60000),
    dict(n=2, period=[1000, 1000], n_push=50, jitter=100),
    dict(n=8, period=[1000] * 8, n_push=5000, jitter=100, slow_worker=7, slow_factor=4, slow_t0=20000,
         slow_t1=120000),
    dict(n=5, period=[900, 1000, 1100, 1300, 1700], n_push=3000, jitter=50, seed=99),
])
def test_schedule_bit_exact_with_oracle(ss, orc, case):
    s, (k1, w1, t1) = ss.ss_schedule(**case)
    k2, w2, t2 = orc.schedule(**case)
    assert s == 0 and np.array_equal(k1, k2) and np.array_equal(w1, w2) and np.array_equal(t1, t2)


def test_detector_matches_oracle(ss, orc):
    rng = np.random.default_rng(3)
    a, b = ss.Detector(8, 3), orc.Detector(8, 3)
    for _ in range(200):
        samples = rng.integers(5, 20, 8).astype(np.float64)
        busy = rng.integers(1000, 5000, 8).astype(np.float64)
        if rng.random() < 0.5:
            busy[7] *= 4
        fa, ca = a.window(samples, busy)
        fb, cb = b.window(samples, busy)
        assert np.array_equal(fa, fb) and ca == cb


def test_greedy_policy(ss):
    # straggler during BSP -> ASP; clean cluster and BSP quota unmet -> back to BSP; otherwise nothing
    assert ss.ss_greedy_decision(ss.SS_BSP, True, False, 10, 100) == ss.SS_ASP
    assert ss.ss_greedy_decision(ss.SS_BSP, False, True, 10, 100) == -1
    assert ss.ss_greedy_decision(ss.SS_ASP, False, True, 10, 100) == ss.SS_BSP
    assert ss.ss_greedy_decision(ss.SS_ASP, False, True, 100, 100) == -1
    assert ss.ss_greedy_decision(ss.SS_ASP, True, False, 10, 100) == -1
