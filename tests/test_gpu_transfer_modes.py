"""The opt-in device-flag transfer pipeline (CLO_TRANSFER=flags: one
persistent gather kernel per step gated by device flags, no per-layer
launches) must give results identical to the default event-ordered one. The
mode is fixed per process, so the check runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = """
from oracle.bind import Oracle
from tests.engine_harness import make_case, run_and_compare
for kw in (dict(), dict(kv_dtype="bf16", d=128, hq=8, hkv=2, n_prompt=400, k=32, sink=4, recent=64),
           dict(policy="prefetch_only"), dict(always_miss=True, retriever="exact"),
           dict(kv_dtype="bf16", d=128, hq=8, hkv=2, n_prompt=400, k=32, interleaved=True),
           dict(kv_dtype="f32", always_miss=True, interleaved=True)):
    run_and_compare(make_case(**kw), Oracle())
print("flags ok")
"""


def test_flag_transfer_pipeline_matches_oracle():
    env = dict(os.environ, CLO_TRANSFER="flags", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "flags ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("variant", ["lsu", "tma", "lite:128,8", "lite:64,8"])
def test_gather_variants_match_oracle(variant):
    """Every engine-gather copy variant (launch_gather_engine picks TMA bulk or
    LSU by host-region size; CLO_GATHER forces one) moves the same rows."""
    env = dict(os.environ, CLO_GATHER=variant, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("flags ok", "variant ok")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stderr[-3000:]
