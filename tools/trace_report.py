#!/usr/bin/env python
"""Summarise SS_TRACE dumps of a multi-GPU run (one CSV per rank, written at ss_destroy).

    SS_TRACE=/path/prefix torchrun ... bench.py ...;  python tools/trace_report.py /path/prefix [--skip N]

Per kernel kind, medians over launches (after skipping the first N of each rank) of:
  wait    CTA 0's start wait (enter -> waited; kernels that wait for a peer phase)
  body    waited (or enter) -> last CTA signals
  endwait signal -> end wait satisfied (kernels that wait for every rank at their end)
  gap     previous launch's last stamp on this rank -> this launch's enter (device idle or launch latency)
  skew    spread over ranks of the enter stamps of the same launch, after removing each rank's median clock offset
          to rank 0 (globaltimer is per GPU)
"""
import csv
import glob
import statistics
import sys


def load(prefix):
    ranks = []
    for path in sorted(glob.glob(prefix + ".rank*.csv"), key=lambda p: int(p.rsplit("rank", 1)[1][:-4])):
        with open(path) as f:
            ranks.append([dict(r, **{k: int(r[k]) for k in ("enter_ns", "waited_ns", "signal_ns", "end_ns")})
                          for r in csv.DictReader(f)])
    return ranks


def main():
    prefix = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 100
    ranks = load(prefix)
    stats = {}
    for rows in ranks:
        prev_end = None
        for i, r in enumerate(rows):
            last = max(r["end_ns"], r["signal_ns"], r["waited_ns"], r["enter_ns"])
            if i >= skip:
                s = stats.setdefault(r["kernel"], {"wait": [], "body": [], "endwait": [], "gap": [], "skew": []})
                start = r["waited_ns"] or r["enter_ns"]
                if r["waited_ns"]:
                    s["wait"].append(r["waited_ns"] - r["enter_ns"])
                s["body"].append(r["signal_ns"] - start)
                if r["end_ns"]:
                    s["endwait"].append(r["end_ns"] - r["signal_ns"])
                if prev_end is not None:
                    s["gap"].append(r["enter_ns"] - prev_end)
            prev_end = last
    n = min(len(r) for r in ranks)
    off = [statistics.median(rows[i]["enter_ns"] - ranks[0][i]["enter_ns"] for i in range(skip, n)) for rows in ranks]
    for i in range(skip, n):
        ent = [rows[i]["enter_ns"] - o for rows, o in zip(ranks, off)]
        stats[ranks[0][i]["kernel"]]["skew"].append(max(ent) - min(ent))
    print(f"{len(ranks)} ranks, {n} launches each, first {skip} skipped; medians in microseconds")
    print(f"{'kernel':12s} {'count':>6s} {'wait':>8s} {'body':>8s} {'endwait':>8s} {'gap':>8s} {'skew':>8s}")
    for k, s in stats.items():
        med = {m: (statistics.median(v) / 1e3 if v else float('nan')) for m, v in s.items()}
        print(f"{k:12s} {len(s['body']):6d} {med['wait']:8.2f} {med['body']:8.2f} {med['endwait']:8.2f} "
              f"{med['gap']:8.2f} {med['skew']:8.2f}")


if __name__ == "__main__":
    main()
