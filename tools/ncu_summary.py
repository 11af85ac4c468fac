#!/usr/bin/env python
"""Condense ncu captures of the bench into committed JSON summaries (profiles/).

    python tools/ncu_summary.py full  <report.ncu-rep> <config> <out.json> [command...]
        per kernel of an `ncu --set full` capture: dram read / write bytes (traffic), duration, DRAM % of peak,
        registers, grid, dynamic shared memory, achieved occupancy, the §8(d) algorithmic bytes of the launch and the
        cold-cache GB/s they imply
    python tools/ncu_summary.py launches <launches.csv> <out.json>
        share of each of the library's kernels in the device time of an `ncu --metrics gpu__time_duration.sum` launch
        list (serialised, cold caches: the SHARE is comparable with the bench's live share, the absolute time is not)
"""
import csv
import io
import json
import re
import subprocess
import sys

CONFIG_P = {"2": 464_154, "3": 25_557_032, "5a": 100_000_000, "5b": 250_000_000, "5c": 500_000_000,
            "5d": 1_000_000_000}
N = 8   # workers (and pushes per window, pulls per window) in the single-GPU bench configs


def algorithmic_bytes(kind: str, P: int) -> int:
    """BSP superstep (n + 4)·4P; ASP window of n pushes and n pulls (4 + 2n)·4P."""
    return (N + 4) * 4 * P if kind == "bsp_update" else (4 + 2 * N) * 4 * P


def raw(report: str) -> list:
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        recs.append(d)
    return recs


def num(d, key):
    unit = d["_units"].get(key, "").split("/")[0]
    v = float(d[key].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
             "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
    return v * scale


def full(report: str, config: str, out: str, command: str):
    P = CONFIG_P[config]
    res = {}
    for d in raw(report):
        name = d["Kernel Name"]
        kind = "bsp_update" if "bsp_update" in name else "asp_replay" if "asp_replay" in name else None
        if kind is None or kind in res:
            continue
        rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
        dur = num(d, "gpu__time_duration.sum")
        alg = algorithmic_bytes(kind, P)
        res[kind] = {"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic": rd + wr,
                     "duration_us": dur,
                     "dram_pct_peak": float(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
                     "regs": int(float(d.get("launch__registers_per_thread", "0"))),
                     "grid": int(float(d.get("launch__grid_size", "0"))),
                     "dyn_smem_per_block_bytes": num(d, "launch__shared_mem_per_block_dynamic")
                     if "launch__shared_mem_per_block_dynamic" in d else None,
                     "achieved_occupancy_pct": float(d.get("sm__warps_active.avg.pct_of_peak_sustained_active",
                                                           "nan")),
                     "algorithmic_bytes": alg, "traffic_over_algorithmic": (rd + wr) / alg,
                     "achieved_GBps_cold": alg / (dur * 1e-6) / 1e9}
    res["command"] = command
    res["note"] = ("cold-cache serialised replay (ncu); traffic = dram read + write per launch; algorithmic bytes per "
                   "SURVEY §8(d) (BSP (n+4)·4P, ASP window (4+2n)·4P, n = 8)")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def launches(path: str, out: str):
    tot, per = 0.0, {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for d in csv.DictReader(io.StringIO("".join(lines))):
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        m = re.search(r"(\w+_kernel)", name)
        short = m.group(1) if m else name
        t = float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
        rec = per.setdefault(short, {"launches": 0, "us": 0.0})
        rec["launches"] += 1
        rec["us"] += t
        tot += t
    res = {k: dict(v, share=v["us"] / tot, avg_us=v["us"] / v["launches"]) for k, v in per.items()}
    res["_total_us"] = tot
    res["_note"] = ("ncu launch list of the bench command (gpu__time_duration.sum, --clock-control none): serialised, "
                    "cold caches; synth_grad launches are the bench's input setup outside the timed region")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4], " ".join(sys.argv[5:]))
    else:
        launches(sys.argv[2], sys.argv[3])
