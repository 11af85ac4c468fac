import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from bench import CONFIGS, SEED
from paper_2104_08364_b200 import syncswitch as ss
cfg = CONFIGS["2"]; P, n, S = cfg["P"], cfg["n"], cfg["S"]
g = ss.SyncSwitch(torch.zeros(P, device="cuda"), S, n, 0.1, 0.9); g.set_window(16)
ring = {(j, r): torch.empty(P, device="cuda") for j in range(n) for r in range(2)}
dst = {j: torch.empty(P, device="cuda") for j in range(n)}
gp = (ctypes.c_void_p * n)(*[ss.ptr(ring[(j, 0)]) for j in range(n)])
ws = np.arange(n, dtype=np.int32); vs = np.zeros(n, dtype=np.int64)
ev = (ss.ss_event * (2 * n))()
for j in range(n):
    ev[2*j] = ss.ss_event(0, j, 0, ss.ptr(ring[(j, 1)]), None); ev[2*j+1] = ss.ss_event(1, j, 0, None, ss.ptr(dst[j]))
L, c = ss.lib, g.ctx
gpc = ctypes.cast(gp, ctypes.c_void_p); evc = ctypes.cast(ev, ctypes.c_void_p)
T = np.zeros(5); ver = 0
N = 3000
for it in range(N + 200):
    vs[:] = ver
    for j in range(n): ev[2*j].version = ver + 1
    t0 = time.perf_counter_ns()
    s = L.ss_bsp_step(c, gpc, ws.ctypes.data, vs.ctypes.data, n)
    t1 = time.perf_counter_ns()
    s |= L.ss_switch(c, 1, 0)
    t2 = time.perf_counter_ns()
    s |= L.ss_asp_replay(c, evc, 2 * n, None)
    t3 = time.perf_counter_ns()
    s |= L.ss_switch(c, 0, 0)
    t4 = time.perf_counter_ns()
    assert s == 0
    ver += 1 + n
    if it >= 200: T += np.array([t1-t0, t2-t1, t3-t2, t4-t3, t4-t0]) / 1e3
print("host us per call: bsp_step %.2f switch(ASP) %.2f asp_replay %.2f switch(BSP, flush) %.2f total %.2f" % tuple(T / N))
# same with a null kernel launch for scale
t0 = time.perf_counter_ns()
x = torch.empty(1, device="cuda")
for _ in range(N): x.add_(1)
print("torch tiny op: %.2f us" % ((time.perf_counter_ns() - t0) / 1e3 / N))
# the pointer classification the library does per event (cudaPointerGetAttributes)
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if cudart is not None:
    buf = ctypes.create_string_buffer(64)
    p = ctypes.c_void_p(ss.ptr(dst[0]))
    t0 = time.perf_counter_ns()
    for _ in range(N):
        cudart.cudaPointerGetAttributes(buf, p)
    print("cudaPointerGetAttributes: %.3f us" % ((time.perf_counter_ns() - t0) / 1e3 / N))
