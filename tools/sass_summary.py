#!/usr/bin/env python
"""SASS evidence for the built library: per-kernel counts of the memory / sync opcodes that show how each kernel moves
data (UBLKCP = cp.async.bulk TMA, SYNCS = mbarrier, LDG/STG .128 = 128-bit vector accesses, .SYS = system-scope
flags over NVLink, multimem stores), plus the instructions around the first UBLKCP of the TMA window kernel.

    python tools/sass_summary.py > profiles/r02_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2104_08364_b200", "libsyncswitch.so")
PREFIXES = ("UBLKCP", "SYNCS", "LDG", "STG", "LDGSTS", "MEMBAR", "ATOMG", "RED", "UTMA", "LDS", "STS", "FFMA",
            "FADD", "MULTIMEM", "UMULTIMEM")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    blocks = sass.split("Function : ")[1:]
    print(f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)} (sm_100a)\n")
    first_bulk = None
    for blk in blocks:
        name = blk.split("\n", 1)[0].strip()
        short = re.sub(r"^_ZN2ss\d+_GLOBAL__N__\w+?_kernels_cu_[0-9a-f]{8}\d+", "", name)
        ops = collections.Counter(
            re.findall(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", blk, re.M))
        keys = sorted(k for k in ops if k.startswith(PREFIXES))
        print(short)
        print("  " + ", ".join(f"{k}:{ops[k]}" for k in keys))
        if first_bulk is None and "asp_replay_tma" in name and "UBLKCP" in blk:
            lines = [ln for ln in blk.splitlines() if re.match(r"^\s+/\*[0-9a-f]+\*/", ln)]
            i = next(k for k, ln in enumerate(lines) if "UBLKCP" in ln)
            first_bulk = (short, lines[max(0, i - 6): i + 4])
    if first_bulk:
        print(f"\n# around the first UBLKCP of {first_bulk[0]}")
        for ln in first_bulk[1]:
            print(re.sub(r"\s+/\* 0x[0-9a-f]+ \*/", "", ln).rstrip())
    return 0


if __name__ == "__main__":
    sys.exit(main())
