"""One rank of the multi-GPU parity run (launched by tests/test_multi_gpu.py through torchrun, one process per GPU).

Runs, through the C-ABI at G ranks: BSP supersteps, an in-place switch, a seeded ASP schedule with pulls, a switch
back and more BSP steps, on synth_grad gradients. Writes the protocol integers, the final parameters and momentum,
and every pull snapshot of the workers hosted here to <out>/rank<r>.npz. The test compares them with the oracle.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2104_08364_b200 import syncswitch as ss  # noqa: E402

SEED = 20241018


def sample_indices(P, count):
    rng = np.random.default_rng(0)
    return np.unique(np.concatenate([rng.choice(P, count - 4, replace=False), [0, 1, P - 2, P - 1]]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--P", type=int, default=100003)
    ap.add_argument("--nworkers", type=int, default=4)
    ap.add_argument("--nshards", type=int, default=4)
    ap.add_argument("--window", type=int, default=7)
    ap.add_argument("--bsp1", type=int, default=3)
    ap.add_argument("--pushes", type=int, default=60)
    ap.add_argument("--bsp2", type=int, default=2)
    ap.add_argument("--fused", type=int, default=-1)
    ap.add_argument("--gbuf", type=int, default=0,
                    help="superstep gradients written into the context's exported gradient buffers (zero copy)")
    ap.add_argument("--drop", type=int, default=-1, help="elastic: worker left out of --bsp-drop BSP steps")
    ap.add_argument("--bsp-drop", type=int, default=0)
    ap.add_argument("--sample", type=int, default=0, help="save only this many sampled elements (full-size runs)")
    ap.add_argument("--host-buffers", type=int, default=0, help="gradients and pull destinations in host memory")
    ap.add_argument("--scenario", type=int, default=-1, help="run ss_scenario_run with this policy instead")
    ap.add_argument("--nesterov", type=int, default=0)
    ap.add_argument("--nan-bsp", type=int, default=0,
                    help="after --bsp1 supersteps, one superstep whose worker-0 gradient is NaN at the last element "
                         "(owned by the last rank); every rank records its ss_sync status")
    ap.add_argument("--capture", type=int, default=-1,
                    help="bench step (BSP + switch + n push/pull + switch) once, captured once, replayed this often")
    ap.add_argument("--capture-bsp-only", type=int, default=0,
                    help="the captured step is one BSP superstep (an odd number of fused exchanges per capture)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P, n, S = a.P, a.nworkers, a.nshards
    hosted = [j for j in range(n) if (j * world) // n == rank]

    w0 = torch.empty(P, device="cuda")
    ss.ss_check(ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0))
    w0.mul_(64.0)
    torch.cuda.synchronize()
    g = ss.SyncSwitch(w0, S, n, 0.1, 0.9)
    uid = [ss.ss_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    g.init_dist(rank, world, uid[0])
    if a.fused >= 0:
        g.set_fused(a.fused)
    if a.nesterov:
        g.set_nesterov(True)
    g.set_window(a.window)
    g.set_lr_schedule([a.bsp1 + 10], [0.5])
    counter = {j: 0 for j in range(n)}
    keep = []

    def grad(j):
        k = counter[j]
        counter[j] += 1
        if j not in hosted:
            return None
        buf = torch.empty(P, device="cuda")
        ss.ss_check(ss.ss_synth_grad(SEED, j, k, 0, P, buf))
        if a.host_buffers:                 # the e2e path: pinned host memory, staged by the library
            torch.cuda.synchronize()
            buf = buf.cpu().pin_memory()
        keep.append(buf)
        return buf

    def bsp_grads(ids):
        """Gradients of one superstep. --gbuf: written in place into ss_grad_buffer (the previous superstep borrowed
        them until ss_sync, so sync first; synth_grad runs on the library's stream behind it)."""
        if not a.gbuf:
            return {j: grad(j) for j in ids}
        g.sync()
        out = {}
        for j in ids:
            k = counter[j]
            counter[j] += 1
            if j in hosted:
                ptr = g.grad_buffer(j)
                ss.ss_check(ss.ss_synth_grad(SEED, j, k, 0, P, ptr, g.stream))
                out[j] = ptr
            else:
                out[j] = None
        return out

    if a.scenario >= 0:
        sc = dict(n_workers=n, batch=128, total_samples=600 * 128, quota_num=1, quota_den=2, period=1000, jitter=0,
                  sched_seed=7, grad_seed=SEED, slow_worker=n - 1, slow_factor=4, slow_t0=3000, slow_t1=30000,
                  window_ticks=4000, K=2, policy=a.scenario)
        s_, log, res = ss.ss_scenario_run(g.ctx, sc)
        ss.ss_check(s_, g.ctx)
        g.sync()
        st = g.stats(64)
        np.savez(os.path.join(a.out, f"rank{rank}.npz"), w=g.params(), v=g.velocity(), log=np.array(log),
                 res=np.array([res[k] for k in ("bsp_steps", "asp_pushes", "dropped", "end_tick", "version")]),
                 hist=st["hist"], plog=g.log())
        g.close()
        dist.barrier()
        dist.destroy_process_group()
        return

    if a.capture >= 0:
        g.set_lr_schedule([1 << 40], [0.5])       # no lr boundary inside the replayed versions
        bsp_g = {j: grad(j) for j in range(n)}
        asp_g = {j: grad(j) for j in range(n)}
        dst = {j: torch.empty(P, device="cuda") for j in hosted}

        def step():
            v = g.version
            g.bsp_step([bsp_g[j] for j in hosted], hosted, [v] * len(hosted))
            if a.capture_bsp_only:
                return
            g.switch(ss.SS_ASP, 0)
            for j in range(n):
                assert g.asp_push(j, asp_g[j], v + 1) == j
                g.pull(j, dst.get(j))
            g.switch(ss.SS_BSP, 0)

        step()
        g.capture_begin()
        step()
        assert g.capture_end() == (1 if a.capture_bsp_only else 1 + n)
        g.capture_replay(a.capture)
        g.sync()
        st = g.stats(64)
        np.savez(os.path.join(a.out, f"rank{rank}.npz"), w=g.params(), v=g.velocity(), log=g.log(), hist=st["hist"],
                 version=st["version"], snaps=np.stack([dst[j].cpu().numpy() for j in hosted]) if hosted else
                 np.zeros((0, P), np.float32), hosted=np.array(hosted))
        g.close()
        dist.barrier()
        dist.destroy_process_group()
        return

    for _ in range(a.bsp1):
        gs = bsp_grads(range(n))
        g.bsp_step([gs[j] for j in hosted], hosted, [g.version] * len(hosted))
    if a.nan_bsp:
        gs = {j: grad(j) for j in range(n)}
        if 0 in hosted:
            gs[0][P - 1] = float("nan")
            torch.cuda.synchronize()
        s1 = g.bsp_step_status([gs[j] for j in hosted], hosted, [g.version] * len(hosted))
        s2 = g.sync_status()                 # collective: every rank must see the divergence here
        s3 = g.bsp_step_status([gs[j] for j in hosted], hosted, [g.version] * len(hosted))   # sticky
        np.savez(os.path.join(a.out, f"rank{rank}.npz"), status=np.array([s1, s2, s3]), hosted=np.array(hosted))
        g.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    if a.drop >= 0:
        members = [j for j in range(n) if j != a.drop]
        g.set_members(members)
        mine = [j for j in hosted if j in members]
        for _ in range(a.bsp_drop):
            gs = {j: grad(j) for j in members}
            g.bsp_step([gs[j] for j in mine], mine, [g.version] * len(mine))
        g.set_members(list(range(n)))
    g.switch(ss.SS_ASP, 0)
    kind, worker, _ = ss.ss_schedule(n, [1000 + 100 * j for j in range(n)], a.pushes, jitter=100, seed=7)[1]
    base, stale, snaps = {}, [], []
    for kd, j in zip(kind, worker):
        j = int(j)
        if kd == 1:
            dst = None
            if j in hosted:
                dst = torch.empty(P, pin_memory=True) if a.host_buffers else torch.empty(P, device="cuda")
            base[j] = g.pull(j, dst)
            if dst is not None:
                snaps.append(dst)
        else:
            stale.append(g.asp_push(j, grad(j), base[j]))
    g.switch(ss.SS_BSP, 0)
    for _ in range(a.bsp2):
        gs = bsp_grads(range(n))
        g.bsp_step([gs[j] for j in hosted], hosted, [g.version] * len(hosted))
    g.sync()
    w = g.params()
    v = g.velocity()
    st = g.stats(64)
    if a.sample:
        idx = sample_indices(P, a.sample)
        ti = torch.from_numpy(idx).cuda()
        w, v = w[idx], v[idx]
        snap_arr = np.stack([s[ti].cpu().numpy() for s in snaps]) if snaps else np.zeros((0, len(idx)), np.float32)
    else:
        snap_arr = np.stack([s.cpu().numpy().copy() for s in snaps]) if snaps else np.zeros((0, P), np.float32)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), w=w, v=v, stale=np.array(stale), log=g.log(),
             hist=st["hist"], version=st["version"], dropped=st["dropped"], snaps=snap_arr,
             hosted=np.array(hosted), nvls=int(g.exchange()["nvls"]))
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
