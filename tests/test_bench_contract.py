"""bench.py's JSON-line contract: the reference arm (CPU oracle, runs here) and
the GPU arm on a small config (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"]


def run_bench(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"], 600)
    for k in BASE_KEYS + ["impl", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench(["--config", "c1", "--steps", "3", "--warmup", "3", "--cpu-seconds", "2"], 900)
    for k in BASE_KEYS + ["roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]:
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["n_gpus"] == 1
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1
    assert cb["single_thread"]["cores"] == 1 and cb["single_thread"]["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_gpu_arm_fp64_roofline_on_c3_clone():
    d = run_bench(["--config", "c3", "--c3-cells", "48", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                   "--no-e2e"], 900)
    r = d["roofline_fp64"]
    assert r is not None and r["bound"] == "alu" and r["unit"] == "TFLOP/s"
    assert 20 < r["peak"] < 60 and 0 < r["frac"] < 1 and r["flops_per_update"] > 300
    assert d["roofline"]["traffic"] > 0 and d["roofline"]["traffic_source"]["kind"].startswith("static")
    # the mover against its binding unit (shared-memory crossbar at the run's clock)
    sm = d["roofline_smem"]
    assert sm is not None and sm["bound"] == "smem" and sm["unit"] == "GB/s"
    assert 0 < sm["frac"] < 1 and abs(sm["frac"] - sm["achieved"] / sm["peak"]) < 1e-9
    assert sm["wavefronts_source"]["kind"].startswith("static")
