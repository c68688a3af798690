"""bench.py's JSON-line contract (the driver parses it): the reference arm on the host (CPU), and
our arm on the GPU -- every key the contract names present and sane."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().split("\n") if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _common(d, steps, warmup):
    assert d["metric"].startswith("verified draft positions/sec")
    assert d["unit"] == "positions/s" and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["higher_is_better"] is True and d["scaling"] in ("strong", "weak")
    assert d["vs_baseline"] is None and d["data"] == "synthetic"
    assert d["config"]["workload"] == "llama2"


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--config", "llama2", "--steps", "1", "--warmup", "3", "--ref-sample", "2"])
    _common(d, 1, 3)
    assert d["impl"] == "reference" and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _line(["--config", "llama2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"])
    _common(d, 3, 3)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2 and r["peak"] > 1000
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] == 3 * 3                      # core, tail, rollback per timed step
    assert d["clocks"]["sm_mhz"] > 0
    assert d["config"]["launch"].startswith("one CUDA graph")
    assert d["timeouts"] == 0
