"""One rank of the multi-GPU protocol fuzz (tests/test_gpu_fuzz.py, launched through torchrun, one process per GPU).

Runs the seeded random program of tests/fuzz_program.py through the C-ABI, SPMD: every rank makes every call, with
gradients and pull destinations only on the rank hosting the worker. Records each call's (status, value), the final
parameters, momentum, protocol integers and the snapshots of the pulls of the workers hosted here, in pull order, to
<out>/rank<r>.npz.
"""
import argparse
import collections
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fuzz_program import Program  # noqa: E402
from paper_2104_08364_b200 import syncswitch as ss  # noqa: E402

SEED = 20241018


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--seed", type=int, required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prog = Program(a.seed, world)
    P, n = prog.P, prog.n
    hosted = [j for j in range(n) if (j * world) // n == rank]

    w0 = torch.empty(P, device="cuda")
    ss.ss_check(ss.ss_synth_grad(SEED + 1, 255, 0, 0, P, w0))
    w0.mul_(64.0)
    torch.cuda.synchronize()
    g = ss.SyncSwitch(w0, prog.S, n, 0.1, 0.9)
    uid = [ss.ss_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    g.init_dist(rank, world, uid[0])
    g.set_fused(prog.fused)
    g.set_window(prog.window)
    g.set_lr_schedule(prog.bounds, prog.factors)
    g.set_lr_policy(prog.asp_rule, prog.lam)
    g.set_nesterov(prog.nesterov)
    k = collections.Counter()
    keep, base, rec, snaps = [], {}, [], {j: [] for j in hosted}

    def grad(j):
        kk = k[j]
        k[j] += 1
        if j not in hosted:
            return None
        d = torch.empty(P, device="cuda")
        ss.ss_check(ss.ss_synth_grad(SEED, j, kk, 0, P, d))
        keep.append(d)
        return d

    for _ in range(prog.n_ops):
        ver = g.version
        op = prog.next_op(g.stats(1)["protocol"], ver, base)
        if op[0] == "bsp":
            js, vers = prog.bsp_call(op, ver, range(n))
            gs = {j: grad(j) for j in js}
            mine = [j for j in js if j in hosted]
            rec.append((g.bsp_step_status([gs[j] for j in mine], mine, [vers[js.index(j)] for j in mine]), 0))
        elif op[0] == "push":
            s, st = g.asp_push_status(op[1], grad(op[1]), op[2])
            rec.append((s, st if s == 0 else 0))
        elif op[0] == "pull":
            dst = torch.empty(P, device="cuda") if op[1] in hosted else None   # SPMD pull rule (header)
            if dst is not None:
                keep.append(dst)       # borrowed: written stream-ordered, valid after ss_sync (SV §8b)
            s, v = ss.ss_pull(g.ctx, op[1], dst)
            base[op[1]] = v
            if dst is not None and op[2]:
                snaps[op[1]].append(dst)
            rec.append((s, v))
        elif op[0] == "switch":
            rec.append((g.switch_status(op[1], op[2]), 0))
        else:
            g.sync()
            rec.append((0, 0))
    g.sync()
    st = g.stats(64)
    out = dict(rec=np.array(rec, np.int64).reshape(-1, 2), w=g.params(), v=g.velocity(), log=g.log(),
               hist=st["hist"], version=st["version"], dropped=st["dropped"], hosted=np.array(hosted, np.int64))
    for j in hosted:
        out[f"snaps{j}"] = (np.stack([d.cpu().numpy() for d in snaps[j]]) if snaps[j]
                            else np.zeros((0, P), np.float32))
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
