"""bench.py's JSON contract (the driver parses it): the reference arm (the CPU oracle) on the toy config runs
here; the GPU arm is checked on the toy config under -m gpu."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_warmup_below_three_is_refused():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode != 0


@pytest.mark.gpu
def test_gpu_arm_json_line():
    d = run_bench("--config", "c1", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["scaling"] == "weak" and d["dtype"] == "bf16"
    assert d["data"] == "synthetic" and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 64 * 128 * 4 + 64 * 8 and d["e2e"]["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "alu") and rf["peak"] > 0 and 0 < rf["frac"] and rf["unit"] in ("GB/s", "TFLOP/s")
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
