"""A trace recorded by the REFERENCE (its SyntheticModel with hot runs +
record_trace + write_trace, width 4) replayed by both engines: the reference
DecodeEngine over its TraceSource, and the CUDA engine over libclo's reader
with f32 KV storage (every value it consumes is bit-identical). The
cache_state_json documents must agree key for key — selections, decisions,
aggregated histories bit-exact — and the outputs within the f32 tolerance."""
import json

import numpy as np
import pytest

from oracle.bind import Reference
from paper_2511_14510_b200 import DecodeEngine, EngineConfig, ModeFlags, ModelShape, PartitionPlan, profiles_from_arrays
from paper_2511_14510_b200.trace import TraceSource
from tests.engine_harness import POLICY_CODE, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not Reference.available(), reason="reference library not built")]


@pytest.mark.parametrize("retriever", ["sign_hash", "exact"])
def test_reference_trace_replays_identically(tmp_path, retriever):
    from oracle.bind import EngineCfg
    L, hq, hkv, d, n, steps, k = 3, 8, 2, 64, 600, 8, 64
    path = tmp_path / "ref.bin"
    ref = Reference()
    ref.record_synthetic_trace(path, L, hq, hkv, d, n, steps, d_model=96, sigma_step=0.05, seed=11, width=4)
    rng = np.random.default_rng(3)
    m = hq // hkv
    qimp = rng.uniform(0, 1, (L, hkv, m))
    tau = rng.uniform(0.5, 0.95, (L, hkv))
    pers = np.zeros((L, hkv), np.int32)
    pers[0] = 1

    cfg = EngineConfig(shape=ModelShape(L, hq, hkv, d, 4), k=k, sink_tokens=4, recent_tokens=64,
                       retriever=retriever, hash_bits=256, retriever_seed=5, policy="similarity",
                       mode=ModeFlags(), collect_outputs=True, batch=1, kv_dtype="f32")
    src = TraceSource(path, kv_dtype="f32")
    eng = DecodeEngine(cfg, profiles_from_arrays(tau, qimp),
                       PartitionPlan(layers=[[g for g in range(hkv) if pers[l, g]] for l in range(L)]), src)
    eng.run()
    got = np.stack(eng.collected_outputs())[:, 0]  # [steps][L][hq][d]
    got_state = json.loads(eng.cache_state_json())

    c = EngineCfg()
    c.num_layers, c.num_q_heads, c.num_kv_heads, c.head_dim, c.bytes_per_element = L, hq, hkv, d, 4
    c.k, c.sink_tokens, c.recent_tokens = k, 4, 64
    c.retriever = 0 if retriever == "exact" else 1
    c.hash_bits, c.retriever_seed, c.policy = 256, 5, POLICY_CODE["similarity"]
    c.n_prompt, c.steps = n, steps
    want, want_json = ref.run_engine_trace(c, tau, qimp, pers, path)
    want_state = json.loads(want_json)

    assert rel_l2(got, want).max() <= 1e-3
    for key in ("hits", "misses", "transferred_bytes", "persistent_served_bytes"):
        assert got_state["totals"][key] == want_state["totals"][key], key
    assert got_state["totals"]["misses"] > 0 and got_state["totals"]["hits"] > 0  # the cache was exercised
    for lg, lw in zip(got_state["layers"], want_state["layers"]):
        for hg, hw in zip(lg["heads"], lw["heads"]):
            assert hg == hw, (lg["layer"], hg["kv_head"])
