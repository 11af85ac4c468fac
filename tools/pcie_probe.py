#!/usr/bin/env python
"""Host<->device copy bandwidth with 1, 2 and 4 GPUs copying at once (pinned memory, 1 GB per GPU per direction):
shows whether GPUs share a PCIe uplink (what bounds the multi-GPU e2e numbers)."""
import itertools
import subprocess
import threading
import time

import torch


def run(devs, direction):
    n = 1 << 28
    host = [torch.empty(n, pin_memory=True) for _ in devs]
    dev = [torch.empty(n, device=f"cuda:{d}") for d in devs]
    streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in devs]

    def go(i):
        with torch.cuda.stream(streams[i]):
            for _ in range(3):
                if direction == "h2d":
                    dev[i].copy_(host[i], non_blocking=True)
                else:
                    host[i].copy_(dev[i], non_blocking=True)
        streams[i].synchronize()

    go_all = lambda: [t.join() for t in [threading.Thread(target=go, args=(i,)) for i in range(len(devs))]
                      if not t.start()]
    go_all()
    t0 = time.perf_counter()
    go_all()
    el = time.perf_counter() - t0
    return 3 * 4 * n * len(devs) / el / 1e9


if __name__ == "__main__":
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
    G = torch.cuda.device_count()
    sets = [[0]] + ([[0, 1]] if G > 1 else []) + ([[0, 2], [0, 3]] if G > 3 else []) + ([list(range(G))] if G > 2 else [])
    for devs, d in itertools.product(sets, ["h2d", "d2h"]):
        print(f"GPUs {devs} {d}: {run(devs, d):7.1f} GB/s total")
