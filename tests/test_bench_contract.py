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


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself
    under torch.distributed.run with 2 ranks (127.0.0.1 rendezvous); rank 0
    alone prints the line, which reports n_gpus == 2. The reference arm runs
    on CPU, so this exercises the launcher here."""
    from oracle.bind import Reference
    if not Reference.available():
        pytest.skip("reference library not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "1", "--ctx", "4096", "--cpu-threads", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


@pytest.mark.gpu
def test_our_arm_two_ranks_same_device():
    """Our arm through the self-launcher: 2 request-sharded ranks on cuda:0
    (functional check of the multi-rank path on a 1-GPU box, not a number)."""
    d = _run(["--gpus", "2", "--same-device", "--steps", "3", "--warmup", "3", "--ctx", "8192", "--batch", "2",
              "--layers", "3", "--no-e2e", "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "request-sharded x2"
