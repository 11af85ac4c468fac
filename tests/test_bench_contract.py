"""bench.py's output contract, checked on the CPU through the reference arm (the oracle): one JSON line with the keys
the driver reads. The GPU arm's line is produced on the B200 (profiles/r01_bench_config3.json)."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--config", "2"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"] and "model" not in d["config"]
    assert set(d["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"} and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]


def test_gpu_line_recorded_with_required_keys():
    """The committed round-2 default line (config 3, 1 GPU) carries every key the contract names, and its numbers are
    internally consistent: roofline fraction = achieved / peak, the dominant kernel's time within a step, the step's
    floor fraction = value / floor."""
    with open(os.path.join(ROOT, "profiles", "r02_bench_config3.json")) as f:
        d = json.loads(f.read().splitlines()[0])
    for k in ("roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "step_floor", "protocol_rates"):
        assert k in d, k
    rf = d["roofline"]
    assert set(rf) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert rf["avg_launch_us"] < 1e3 * d["ms_per_step"]
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    fl = d["step_floor"]
    assert abs(fl["frac_of_floor"] - d["value"] / fl["steps_per_s_at_peak"]) < 1e-6 and fl["frac_of_floor"] <= 1.0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


def test_multi_gpu_self_launch_command(monkeypatch):
    """`python bench.py --gpus N` from a plain shell starts its own N ranks (torch.distributed.run, 127.0.0.1); under
    torchrun (WORLD_SIZE set) it runs as the rank it is."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "20", "--warmup", "5"])
    a = bench.parse()
    assert bench._self_launch(a) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-6:] == ["--gpus", "4", "--steps", "20", "--warmup", "5"]
    assert cmd[-7].endswith("bench.py")


def test_step_floor_values():
    """The per-N floor the bench line reports next to its value (SURVEY §8(d) bytes per unit), against hand values:
    config 3 (P = 25,557,032, S = n = 8; P_pad = 25,557,248) at G = 2: 2 * 1/2 * 4 * P_pad * (1 + 8/2) = 511.1 MB per
    GPU per direction -> 1,760.8 steps/s at 900 GB/s; at G = 4: 2 * 3/4 * 4 * P_pad * 3 = 460.0 MB -> 1,956.4; one GPU:
    (3 * 8 + 8) * 4 * P = 3.271 GB at 6,543.1 GB/s -> 2,000.2 steps/s."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    P, S, n = 25_557_032, 8, 8
    f2 = bench.step_floor(2, P, S, n, 1000.0, 6543.1)
    assert abs(f2["bytes_per_gpu_per_direction"] - 511_144_960) < 1 and abs(f2["steps_per_s_at_peak"] - 1760.75) < 0.01
    f4 = bench.step_floor(4, P, S, n, 1000.0, 6543.1)
    assert abs(f4["bytes_per_gpu_per_direction"] - 460_030_464) < 1 and abs(f4["steps_per_s_at_peak"] - 1956.39) < 0.01
    f1 = bench.step_floor(1, P, S, n, 1000.0, 6543.1)
    assert f1["bytes"] == 32 * 4 * P and abs(f1["steps_per_s_at_peak"] - 2000.15) < 0.01
    assert abs(f1["frac_of_floor"] - 1000.0 / f1["steps_per_s_at_peak"]) < 1e-12
