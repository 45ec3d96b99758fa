"""bench.py's JSON line keeps the driver's contract (one line, every key the
task names, consistent units), on a short run of the real config-2 bench."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "4"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["unit"] == "frames/s" and d["higher_is_better"] is True and d["value"] > 0
    assert abs(d["value"] - 1000.0 / d["ms_per_step"]) / d["value"] < 1e-6
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "frames/s"
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] >= 100 * d["steps"]
    c = d["clocks"]
    assert "sm_mhz" in c and "reasons" in c


@pytest.mark.parametrize("mode", [["--mode", "rows"], ["--shard-encoder"], ["--mode", "frames"]])
def test_bench_other_partitions_single_gpu(mode):
    """The N > 1 partitions' code paths at N = 1 (rows: the band render and
    the band gather; --shard-encoder: encode_device + the NULL-encoder
    forward; frames: the config-4 video): one valid JSON line each, with the
    pipelined e2e (upload / read-back streams, two frames in flight)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "4"] + mode,
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 100 * d["steps"]
