"""The C-ABI's error contract on the GPU (SURVEY §8(b) conventions: "Errors never partially apply. A rejected push
does not bump the version"): a push or pull rejected while staging its host buffer — during a graph
capture (SS_E_STATE) or when the staging allocation fails (SS_E_OOM) — leaves the version, the staleness histogram,
the applied-update log and the worker's base version exactly as they were, and the context keeps working: the same
call succeeds afterwards and the run stays bit-identical to the oracle's run of the accepted calls only.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 20241018
BSP, ASP = 0, 1
SS_E_STATE, SS_E_OOM = 2, 9


@pytest.fixture(scope="module")
def ss():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2104_08364_b200 import build
    build.build()
    from paper_2104_08364_b200 import syncswitch
    torch.cuda.init()
    return syncswitch


def _state(g):
    st = g.stats(64)
    return st["version"], st["hist"].copy(), st["dropped"], g.log().copy()


def _same(a, b):
    return a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2] and np.array_equal(a[3], b[3])


def _setup(ss, orc, P, n, S):
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    g = ss.SyncSwitch(torch.from_numpy(w0).cuda(), S, n, 0.1, 0.9)
    o = orc.Oracle(w0, S, n, 0.1, 0.9)
    gb = [orc.synth_grad(SEED, j, 0, 0, P) for j in range(n)]
    dg = [torch.from_numpy(x).cuda() for x in gb]
    g.bsp_step(dg)
    g.flush()                                               # issue the (deferred) superstep while dg is alive
    g.sync()
    assert o.bsp_step(gb) == 0
    g.switch(ASP, 0)
    o.switch(ASP, 0)
    return g, o


def test_rejected_calls_during_capture_change_nothing(ss, orc):
    P, n, S = 4099, 2, 2
    g, o = _setup(ss, orc, P, n, S)
    h = orc.synth_grad(SEED, 0, 1, 0, P)                    # host (pageable) gradient
    hdst = np.zeros(P, np.float32)                          # host pull destination
    before = _state(g)
    g.capture_begin()
    s, st = g.asp_push_status(0, h, 1)
    assert s == SS_E_STATE and st == -1                     # staleness_out untouched
    s, ver = ss.ss_pull(g.ctx, 0, hdst)
    assert s == SS_E_STATE
    s = g.bsp_step_status([h], [0], [1])                    # (also wrong protocol: rejected before anything)
    assert s != 0
    g.capture_end()
    assert _same(_state(g), before)
    # the context is intact: the same calls succeed now, with the staleness the untouched state implies
    assert g.asp_push(0, h, 1) == 0                         # base of worker 0 is still version 1
    assert g.pull(0, hdst) == 2
    assert g.asp_push(1, torch.from_numpy(orc.synth_grad(SEED, 1, 1, 0, P)).cuda(), 1) == 1
    assert o.asp_push(0, h, 1) == (0, 0)
    _, snap, v = o.pull(0)
    assert v == 2 and o.asp_push(1, orc.synth_grad(SEED, 1, 1, 0, P), 1) == (0, 1)
    g.sync()
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.velocity(), o.velocity())
    assert np.array_equal(hdst, snap)
    assert np.array_equal(g.log(), o.log())
    g.close()


def test_rejected_calls_on_staging_oom_change_nothing(ss, orc):
    """Forced staging failure: device memory is exhausted (a torch allocation holds everything but a few MiB) so the
    library's staging-slot cudaMalloc for a host gradient / host pull destination fails."""
    P, n, S = 4_000_003, 2, 2                               # 16 MB staging slots
    g, o = _setup(ss, orc, P, n, S)
    g.sync()
    h = orc.synth_grad(SEED, 0, 1, 0, P)
    hdst = np.zeros(P, np.float32)
    before = _state(g)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    hog = None
    for leave in (4 << 20, 8 << 20, 16 << 20, 64 << 20):
        try:
            hog = torch.empty(free - leave, dtype=torch.uint8, device="cuda")
            break
        except RuntimeError:
            continue
    assert hog is not None
    try:
        s, st = g.asp_push_status(0, h, 1)
        assert s == SS_E_OOM and st == -1, (s, g.last_error())
        s, _ = ss.ss_pull(g.ctx, 1, hdst)
        assert s == SS_E_OOM, (s, g.last_error())
        assert _same(_state(g), before)
    finally:
        del hog
        torch.cuda.empty_cache()
    # memory back: the same calls succeed; nothing of the rejected ones was applied
    assert g.asp_push(0, h, 1) == 0
    assert g.pull(1, hdst) == 2
    assert o.asp_push(0, h, 1) == (0, 0)
    _, snap, _ = o.pull(1)
    g.sync()
    assert np.array_equal(hdst, snap)
    assert np.array_equal(g.params(), o.params()) and np.array_equal(g.log(), o.log())
    g.close()


def test_rejected_push_under_bsp_counts_drop_only(ss, orc):
    """A late push after ASP -> BSP is rejected (SS_E_STATE) and counted as dropped — and nothing else."""
    P, n, S = 1031, 2, 2
    g, o = _setup(ss, orc, P, n, S)
    gd = torch.from_numpy(orc.synth_grad(SEED, 0, 1, 0, P)).cuda()
    g.switch(BSP, 0)
    o.switch(BSP, 0)
    v0, h0, d0, l0 = _state(g)
    s, st = g.asp_push_status(0, gd, 1)
    assert s == SS_E_STATE and st == -1
    v1, h1, d1, l1 = _state(g)
    assert (v1, d1) == (v0, d0 + 1) and np.array_equal(h0, h1) and np.array_equal(l0, l1)
    assert o.asp_push(0, orc.synth_grad(SEED, 0, 1, 0, P), 1)[0] == SS_E_STATE
    assert o.stats()["dropped"] == d1
    g.close()


def test_flush_and_grad_buffer_contract(ss, orc):
    """ss_flush issues pending work without changing protocol state and is a no-op on an empty window; it returns
    SS_E_DIVERGED (sticky) once a non-finite value was produced. ss_grad_buffer exists only in fused multi-GPU mode:
    SS_E_STATE on one GPU, SS_E_INVAL for a bad worker or null output."""
    P, n, S = 1000, 2, 2
    g, o = _setup(ss, orc, P, n, S)
    before = _state(g)
    assert ss.lib.ss_flush(g.ctx) == 0 and _same(_state(g), before)          # nothing pending
    h = torch.from_numpy(orc.synth_grad(SEED, 1, 1, 0, P)).cuda()
    assert g.asp_push(1, h, 1) == 0                                          # staleness 0: deferred in the window
    mid = _state(g)
    assert ss.lib.ss_flush(g.ctx) == 0 and _same(_state(g), mid)             # issued, state unchanged
    assert o.asp_push(1, orc.synth_grad(SEED, 1, 1, 0, P), 1)[0] == 0
    g.sync()
    assert np.array_equal(g.params(), o.params())
    import ctypes
    out = ctypes.c_void_p()
    assert ss.lib.ss_grad_buffer(g.ctx, 0, ctypes.byref(out)) == SS_E_STATE  # single GPU
    assert ss.lib.ss_grad_buffer(g.ctx, 5, ctypes.byref(out)) == 1            # SS_E_INVAL: worker out of range
    assert ss.lib.ss_grad_buffer(g.ctx, 0, None) == 1                         # SS_E_INVAL: null output
    bad = torch.full((P,), float("inf"), device="cuda")
    g.asp_push(0, bad, 2)
    g.flush()
    assert g.sync_status() == 6                                               # SS_E_DIVERGED
    assert ss.lib.ss_flush(g.ctx) == 6                                        # sticky
    g.close()
