"""Pins the C restatement (oracle/clo_oracle.c) to the UNMODIFIED reference
library compiled in place (oracle/_ref/libkvsim_ref.so): bit-identical outputs
on seeded random inputs, op by op and for whole DecodeEngine runs. CPU only;
skipped when the reference could not be built."""
import json

import numpy as np
import pytest

from oracle.bind import OracleError
from tests.engine_harness import make_case, oracle_cfg


def test_rng_streams_identical(oracle, reference):
    for seed in (0, 1, 12345, 2**63 + 7):
        assert np.array_equal(oracle.fill_normal(seed, 4097), reference.fill_normal(seed, 4097))
    for args in ((1, 0, 0), (1, 3, 7), (99, 31, 5)):
        assert oracle.mix_seed3(*args) == reference.mix_seed3(*args)


@pytest.mark.parametrize("variant", [0, 1])
def test_retrieve_scored_bit_exact(oracle, reference, variant):
    rng = np.random.default_rng(variant)
    for trial in range(30):
        n, d = int(rng.integers(40, 400)), int(rng.choice([8, 16, 32, 128]))
        k = int(rng.integers(1, n))
        keys = rng.standard_normal((n, d))
        if trial % 3 == 0:  # tie-heavy: duplicated rows and integer values
            keys = np.round(keys * 2) / 2
            keys[n // 2:] = keys[: n - n // 2]
        q = rng.standard_normal(d)
        a = oracle.retrieve_scored(q, keys, k, variant=variant, seed=trial)
        b = reference.retrieve_scored(q, keys, k, variant=variant, seed=trial)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_encode_bit_exact(oracle, reference):
    rng = np.random.default_rng(9)
    for bits in (8, 64, 128, 256, 512):
        keys = rng.standard_normal((50, 24))
        p1, b1 = oracle.encode_sign_hash(keys, bits, bits)
        p2, b2 = reference.encode_sign_hash(keys, bits, bits)
        assert np.array_equal(p1, p2) and np.array_equal(b1, b2)


def test_merge_bit_exact(oracle, reference):
    rng = np.random.default_rng(3)
    for _ in range(100):
        m = int(rng.integers(1, 6))
        props = []
        for _ in range(m):
            size = int(rng.integers(1, 20))
            idx = rng.choice(40, size, replace=False)
            sc = rng.integers(0, 5, size).astype(float)  # many ties
            props.append(list(zip(map(int, idx), map(float, sc))))
        union = len({i for p in props for i, _ in p})
        k = int(rng.integers(1, union + 1))
        assert np.array_equal(oracle.merge_group_topk(props, k), reference.merge_group_topk(props, k))


def test_lookup_and_attention_bit_exact(oracle, reference):
    rng = np.random.default_rng(5)
    for _ in range(100):
        m, d = int(rng.integers(1, 6)), int(rng.integers(1, 40))
        labels = rng.standard_normal((m, d))
        valid = (rng.random(m) > 0.1).astype(np.int32)
        q = labels + 0.5 * rng.standard_normal((m, d))
        w = rng.uniform(0, 1, m)
        tau = float(rng.uniform(-1, 1))
        a = oracle.lookup(labels, valid, q, w, tau)
        b = reference.lookup(labels, valid, q, w, tau)
        assert a[0] == b[0] and a[1] == b[1] and a[3] == b[3]
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[4], b[4]) and np.array_equal(a[5], b[5])
        n = int(rng.integers(1, 60))
        keys, vals = rng.standard_normal((n, d)), rng.standard_normal((n, d))
        idx = rng.choice(n, int(rng.integers(1, n + 1)), replace=False)
        assert np.array_equal(oracle.topk_attention(q[0], keys, vals, idx),
                              reference.topk_attention(q[0], keys, vals, idx))


def test_host_functions_bit_exact(oracle, reference):
    rng = np.random.default_rng(8)
    for s in np.linspace(0, 1, 41):
        assert oracle.compute_threshold(s, 0.8, 3.0) == reference.compute_threshold(s, 0.8, 3.0)
    for _ in range(50):
        diff = rng.uniform(-1, 1, (4, 8))
        args = dict(t_comp_s=float(rng.uniform(1e-6, 1e-3)), pcie_bw=2e10,
                    mem_head_bytes=float(rng.uniform(1e5, 1e7)), persist_bytes_per_head=1000,
                    hbm_budget_bytes=int(rng.choice([0, 8000, 12000, 20000])))
        a = oracle.plan_partition(diff, **args)
        b = reference.plan_partition(diff, **args)
        assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]
    for n in (1, 3, 4, 10, 67, 68, 69, 1000):
        for sink, recent in ((4, 64), (0, 64), (4, 0), (2, 8)):
            a = oracle.sink_recent_indices(n, sink, recent)
            b = reference.sink_recent_indices(n, sink, recent)
            assert np.array_equal(a[0], b[0]) and a[1] == b[1]


ENGINE_CASES = [
    dict(retriever="exact", always_miss=True, L=4, d=32, n_prompt=160, steps=20, k=13, sink=4,
         recent=64),                                                    # acceptance criterion 4
    dict(retriever="sign_hash"),
    dict(retriever="sign_hash", kv_dtype="bf16", tau=-1.0),
    dict(retriever="exact", always_hit=True),
    dict(retriever="sign_hash", policy="prefetch_only"),
    dict(retriever="sign_hash", tau_override=0.97, persistent=np.array([[1, 0], [0, 1], [0, 0]])),
]


@pytest.mark.parametrize("kw", ENGINE_CASES)
def test_engine_run_bit_exact(oracle, reference, kw):
    case = make_case(batch=1, **kw)
    wl = case["wl"]
    pk, pv, tq, aq, nk, nv = wl.oracle_inputs(0)
    c = oracle_cfg(case)
    outs, js, _ = reference.run_engine(c, case["tau"], case["qimp"], case["persistent"], pk, pv, tq, aq,
                                       nk, nv)
    e = oracle.engine(c, case["tau"], case["qimp"], case["persistent"], pk, pv)
    e.prefill(tq[0])
    for t in range(1, wl.steps + 1):
        got = e.decode_step(tq[t], aq[t], nk[t - 1], nv[t - 1])
        assert np.array_equal(got, outs[t - 1]), f"outputs differ at step {t}"
    doc = json.loads(js)
    s = case["cfg"].shape
    for l in range(s.num_layers):
        for g in range(s.num_kv_heads):
            h = doc["layers"][l]["heads"][g]
            st = e.head_state(l, g)
            assert h["hits"] == st["hits"] and h["misses"] == st["misses"]
            assert h["transferred_bytes"] == st["transferred_bytes"]
            assert h["persistent_served_bytes"] == st["persistent_served_bytes"]
            assert (h["placement"] == "persistent") == st["persistent"]
            if h["placement"] == "offloaded":
                assert h["window_held_tokens"] == st["window_held_tokens"]
                if "entry_indices" in h:
                    assert h["entry_indices"] == list(map(int, st["entry_indices"]))
                    assert h["entry_last_update_step"] == st["entry_last_update_step"]
                    assert h["labels_valid"] == st["labels_valid"]
                    assert h["aggregated_history"] == list(map(float, st["aggregated_history"]))


def test_engine_errors_match(oracle, reference):
    case = make_case(batch=1, steps=2)
    wl = case["wl"]
    pk, pv, tq, aq, nk, nv = wl.oracle_inputs(0)
    c = oracle_cfg(case)
    c.k = wl.n_prompt + 1  # k exceeds the prompt
    with pytest.raises(OracleError) as a:
        oracle.engine(c, case["tau"], case["qimp"], case["persistent"], pk, pv)
    with pytest.raises(OracleError) as b:
        reference.run_engine(c, case["tau"], case["qimp"], case["persistent"], pk, pv, tq, aq, nk, nv)
    assert a.value.code == b.value.code == 2
