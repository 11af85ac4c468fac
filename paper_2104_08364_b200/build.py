"""Builds libsyncswitch.so in-tree with nvcc for sm_100a (the C-ABI of include/syncswitch.h).

    python -m paper_2104_08364_b200.build          # incremental
    python -m paper_2104_08364_b200.build --force
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsyncswitch.so")
SOURCES = ["runtime.cu", "kernels.cu", "control.cpp", "scenario.cpp", "nvls.cpp"]
HEADERS_EXTRA = ["plan.h"]
HEADERS = ["internal.h", "plan.h", "nvls.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """NCCL headers/library shipped with torch's CUDA wheels (the same libnccl.so.2 torch loads)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("NCCL headers / libnccl.so.2 not found in the nvidia wheels")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "syncswitch.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Builds the library (out/defines: tuning variants for tools/kernel_sweep.py; the product is the default)."""
    if out is None and not (force or _stale()):
        return LIB
    inc, lib = nccl_dirs()
    target = out or LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           *[f"-D{d}" for d in defines],
           *[os.path.join(CSRC, s) for s in SOURCES],
           f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}",
           "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
