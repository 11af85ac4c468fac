"""The oracle on seeded random call programs (tests/fuzz_program.py), against invariants the method fixes (CPU).

For every call of every program: version accounting (S:180 — the version grows by exactly one per accepted BSP
superstep and per accepted push, and never otherwise), staleness = version at apply − the version the push was based
on (reading C5), a pull reports the current version, a rejected call changes nothing (SV §8b: errors
never partially apply), pushes rejected under BSP are the dropped ones (reading C8), and the histogram and log
hold exactly the accepted updates (one staleness-0 record per BSP worker, one record per push).
"""
import collections

import numpy as np
import pytest

from fuzz_program import BSP, Program

SEED = 20241018
OK, E_STATE = 0, 2


@pytest.mark.parametrize("case_seed", list(range(40)))
def test_random_programs_keep_the_protocol_invariants(orc, case_seed):
    prog = Program(3000 + case_seed)
    P, n = prog.P, prog.n
    w0 = orc.synth_grad(SEED + 1, 255, 0, 0, P) * np.float32(64.0)
    o = orc.Oracle(w0, prog.S, n, 0.1, 0.9)
    o.set_lr_schedule(prog.bounds, prog.factors)
    o.set_lr_policy(prog.asp_rule, prog.lam)
    o.set_nesterov(prog.nesterov)
    k = collections.Counter()
    base = {}
    accepted_bsp = accepted_push = dropped = 0
    records = []                                   # (staleness) of every accepted update, in order

    def grad(j):
        h = orc.synth_grad(SEED, j, k[j], 0, P)
        k[j] += 1
        return h

    for _ in range(prog.n_ops):
        ver = o.version
        before = (o.params(), o.velocity()) if P <= 4099 else None
        op = prog.next_op(o.stats(1)["protocol"], ver, base)
        s = OK
        if op[0] == "bsp":
            js, vers = prog.bsp_call(op, ver, range(n))
            s = o.bsp_step([grad(j) for j in js], js, vers)
            if s == OK:
                accepted_bsp += 1
                records += [0] * n
                assert o.version == ver + 1
        elif op[0] == "push":
            s, st = o.asp_push(op[1], grad(op[1]), op[2])
            if s == OK:
                accepted_push += 1
                assert st == ver - op[2] >= 0
                records.append(st)
                assert o.version == ver + 1
            elif s == E_STATE:
                dropped += 1
        elif op[0] == "pull":
            s, _, v = o.pull(op[1])
            assert s == OK and v == ver
            base[op[1]] = v
        elif op[0] == "switch":
            s = o.switch(op[1], op[2])
        if s != OK:
            assert o.version == ver
            if before is not None:
                assert np.array_equal(o.params(), before[0]) and np.array_equal(o.velocity(), before[1])
    st = o.stats(256)
    assert st["version"] == accepted_bsp + accepted_push
    assert st["dropped"] == dropped
    hist = np.bincount(np.array(records, np.int64), minlength=256)[:256] if records else np.zeros(256, np.int64)
    assert np.array_equal(np.asarray(st["hist"], np.int64), hist)
    log = o.log()
    assert log.shape[0] == len(records) and np.array_equal(log[:, 2], np.array(records, np.int64).reshape(-1))
    assert np.all(log[:, 3] - log[:, 1] == log[:, 2])           # staleness = version at apply - base version
    o.close()


def test_programs_are_deterministic():
    a, b = Program(77, 2), Program(77, 2)
    assert (a.n, a.S, a.P, a.window, a.fused, a.bounds) == (b.n, b.S, b.P, b.window, b.fused, b.bounds)
    state = (BSP, 5, {0: 3})
    assert [a.next_op(*state) for _ in range(50)] == [b.next_op(*state) for _ in range(50)]
    assert a.S % 2 == 0                             # shards split evenly over the ranks
