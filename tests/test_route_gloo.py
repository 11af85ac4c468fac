"""Multi-rank host logic of the N > 1 path on CPU: world-size 2, 4 and 8 processes over torch.distributed 'gloo'.

Each rank computes its own routing plan with the library's ss_route_plan (the plan.h code the runtime executes with
NCCL or fused NVLink stores), the ranks cross-check that every send has its matching receive, then EXECUTE the plan
with gloo send/recv on CPU tensors carrying position-coded payloads, and verify that every push's gradient slice
lands at its owner and every pull assembles the full parameter vector. No GPU involved.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _grad_val(win, ev, idx):
    return win * 1_000_000 + ev * 10_000 + idx


def _rank_main(rank, world, port, cfg, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2104_08364_b200 import syncswitch as ss
        n, S, P, win, fused = cfg["n"], cfg["S"], cfg["P"], cfg["window"], cfg["fused"]
        st, (kind, worker, _) = ss.ss_schedule(n, [1000 + 37 * j for j in range(n)], cfg["pushes"], jitter=100,
                                               seed=11)
        assert st == 0
        st, ops, nwin = ss.ss_route_plan(rank, world, n, S, P, win, fused, kind, worker)
        assert st == 0
        plans = [None] * world
        dist.all_gather_object(plans, (nwin, ops))
        # 1. every rank cut the sequence into the same windows; sends and receives pair up in order
        assert len({p[0] for p in plans}) == 1
        for a in range(world):
            for b in range(world):
                if a == b:
                    continue
                sends = [o[:2] + o[4:] for o in plans[a][1] if o[2] == 0 and o[3] == b]
                recvs = [o[:2] + o[4:] for o in plans[b][1] if o[2] == 1 and o[3] == a]
                assert sends == recvs, (a, b)
        # 2. execute with gloo and check the data lands where the protocol needs it
        host = lambda j: (j * world) // n  # noqa: E731
        # window-relative event -> (kind, worker), rebuilt from the plan's window cut of this sequence
        events, cur = [], []
        seen_pull = set()
        for kd, wk in zip(kind, worker):
            if len(cur) >= win or (fused and kd == 1 and int(wk) in seen_pull):
                events.append(cur)
                cur, seen_pull = [], set()
            cur.append((int(kd), int(wk)))
            if kd == 1:
                seen_pull.add(int(wk))
            if len(cur) >= win:
                events.append(cur)
                cur, seen_pull = [], set()
        if cur:
            events.append(cur)
        assert len(events) == nwin
        pad = ((P + S - 1) // S + 31) // 32 * 32
        reg = pad * S // world
        lo, hi = min(rank * reg, P), min((rank + 1) * reg, P)
        idx = torch.arange(P, dtype=torch.int64)
        for w in range(nwin):
            wops = [o for o in ops if o[0] == w]
            for phase in (0, 1):
                reqs, checks = [], []
                for (_, ph, op, peer, ev, off, cnt) in wops:
                    if ph != phase:
                        continue
                    tag = phase * 1000 + ev
                    if phase == 0:       # gradient slice of push `ev`: pusher -> owner
                        if op == 0:
                            buf = _grad_val(w, ev, idx[off:off + cnt])
                            reqs.append(dist.isend(buf.contiguous(), peer, tag=tag))
                        else:
                            buf = torch.empty(cnt, dtype=torch.int64)
                            reqs.append(dist.irecv(buf, peer, tag=tag))
                            assert (off, off + cnt) == (lo, hi)
                            checks.append((buf, _grad_val(w, ev, idx[lo:hi])))
                    else:                # snapshot slice of pull `ev`: owner -> puller
                        if op == 0:
                            buf = -_grad_val(w, ev, idx[off:off + cnt])
                            assert (off, off + cnt) == (lo, hi)
                            reqs.append(dist.isend(buf.contiguous(), peer, tag=tag))
                        else:
                            buf = torch.empty(cnt, dtype=torch.int64)
                            reqs.append(dist.irecv(buf, peer, tag=tag))
                            checks.append((buf, -_grad_val(w, ev, idx[off:off + cnt])))
                for r in reqs:
                    r.wait()
                for got, want in checks:
                    assert torch.equal(got, want)
            # coverage: each hosted pull receives every owner region except its own
            for k, (kd, wk) in enumerate(events[w]):
                if kd == 1 and host(wk) == rank:
                    got = sorted((o[5], o[6]) for o in wops if o[1] == 1 and o[4] == k)
                    cover = sorted(got + ([(lo, hi - lo)] if hi > lo else []))
                    pos = 0
                    for off, cnt in cover:
                        assert off == pos
                        pos += cnt
                    assert pos == P
                if kd == 0 and host(wk) != rank and hi > lo:
                    assert any(o[1] == 0 and o[2] == 1 and o[4] == k for o in wops)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("P", [1003, 33])
def test_route_plan_gloo(world, fused, P):
    from paper_2104_08364_b200 import build
    build.build()
    cfg = dict(n=8, S=8, P=P, window=7, fused=fused, pushes=40)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert out[r] == "ok", out[r]
