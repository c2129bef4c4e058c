"""The driver-facing bench.py contract: one JSON line with the keys the
driver reads. CPU: the reference arm (the compiled reference engine on the
host cores) at a tiny context. GPU: our arm at a tiny configuration, with
the roofline / cpu_baseline / e2e / clocks / gpu_launches objects."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle.bind import Reference
    if not Reference.available():
        pytest.skip("reference library not built")
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ctx", "4096", "--cpu-threads", "2"])
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "dtype",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "4", "--warmup", "3", "--ctx", "8192", "--batch", "2", "--layers", "4",
              "--cpu-threads", "2"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "layer_timing"):
        assert k in d, k
    assert d["steps"] == 4 and d["warmup"] == 3 and d["value"] > 0
    roof = d["roofline"]
    assert roof["bound"] in ("pcie", "hbm", "tensor") and 0 < roof["frac"] <= 1.5 and roof["peak"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 4 * d["kernels_per_step"]
    assert d["cpu_baseline"]["value"] > 0
