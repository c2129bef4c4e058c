"""Pins the C oracle (clo_oracle.c) to the reference's own known-answer tests.

Each case re-expresses a doctest case of /root/reference/proj/tests/unit/*
(doctest is absent, so they cannot be run as shipped); the citation names the
reference file:line. CPU only.
"""
import math

import numpy as np
import pytest

from oracle.bind import OracleError


# ----------------------------------------------------------- attention_test.cpp

def test_single_token_returns_value_row(oracle):  # attention_test.cpp:29-38
    k = np.array([[2.0, 0, 0]])
    v = np.array([[5.0, -1.0, 0.25]])
    out = oracle.topk_attention([1.0, 0, 0], k, v, [0])
    assert list(out) == [5.0, -1.0, 0.25]


def test_uniform_scores_average_values(oracle):  # attention_test.cpp:40-52
    k = np.zeros((3, 4))
    k[0, 1], k[1, 2], k[2, 3] = 1.0, 1.0, -2.0
    v = np.array([[r * 10.0 + c for c in range(4)] for r in range(3)])
    out = oracle.topk_attention([3.0, 0, 0, 0], k, v, [0, 1, 2])
    assert np.allclose(out, [10.0 + c for c in range(4)], rtol=1e-12, atol=0)


def test_basis_vector_topk(oracle):  # attention_test.cpp:94-99
    k = np.eye(4)
    assert list(oracle.topk_select_exact([0, 1.0, 0, 0], k, 1)) == [1]


def test_topk_ties_toward_lower_index(oracle):  # attention_test.cpp:119-131
    k = np.zeros((5, 2))
    k[:, 0] = [0.5, 1.0, 2.0, 1.0, 0.5]
    q = [1.0, 0.0]
    assert list(oracle.topk_select_exact(q, k, 2)) == [1, 2]
    assert list(oracle.topk_select_exact(q, k, 3)) == [1, 2, 3]
    assert list(oracle.topk_select_exact(q, k, 4)) == [0, 1, 2, 3]


def test_topk_rejects_out_of_range_k(oracle):  # attention_test.cpp:133-138
    k = np.zeros((4, 2))
    for bad in (0, 5):
        with pytest.raises(OracleError) as e:
            oracle.topk_select_exact([1.0, 0.0], k, bad)
        assert e.value.code == 2


def test_topk_equals_full_sort(oracle):  # attention_test.cpp:110-117
    rng = np.random.default_rng(4)
    for _ in range(50):
        k = rng.standard_normal((64, 8))
        q = rng.standard_normal(8)
        scores = k @ q
        want = sorted(sorted(range(64), key=lambda i: (-scores[i], i))[:6])
        assert list(oracle.topk_select_exact(q, k, 6)) == want


def test_one_index_returns_row(oracle):  # attention_test.cpp:150-158
    rng = np.random.default_rng(6)
    k, v, q = rng.standard_normal((10, 4)), rng.standard_normal((10, 4)), rng.standard_normal(4)
    assert np.array_equal(oracle.topk_attention(q, k, v, [7]), v[7])


def test_attention_rejects_bad_index_sets(oracle):  # attention_test.cpp:170-179
    k, v = np.zeros((4, 2)), np.zeros((4, 2))
    codes = []
    for idx in ([4], [1, 1]):
        with pytest.raises(OracleError) as e:
            oracle.topk_attention([1.0, 0.0], k, v, idx)
        codes.append(e.value.code)
    assert codes == [4, 2]  # IndexError, ArgumentError
    k[0, 0] = np.nan
    with pytest.raises(OracleError) as e:
        oracle.topk_attention([1.0, 0.0], k, v, [1])
    assert e.value.code == 3  # NumericError (check_qkv scans every row)


def test_attention_matches_long_double_reference(oracle):  # attention_test.cpp:54-64
    rng = np.random.default_rng(1)
    for _ in range(20):
        k, v, q = rng.standard_normal((8, 4)), rng.standard_normal((8, 4)), rng.standard_normal(4)
        s = (k @ q) / math.sqrt(4)
        w = np.exp(s - s.max())
        want = (w / w.sum()) @ v
        out = oracle.topk_attention(q, k, v, list(range(8)))
        assert np.linalg.norm(out - want) / np.linalg.norm(want) < 1e-6


def test_window_arithmetic(oracle):  # attention_test.cpp:181-200
    idx, cl = oracle.sink_recent_indices(100, 4, 64)
    assert not cl and list(idx) == list(range(4)) + list(range(36, 100))
    idx, _ = oracle.sink_recent_indices(100, 0, 64)
    assert idx[0] == 36 and idx[-1] == 99 and len(idx) == 64
    idx, cl = oracle.sink_recent_indices(10, 4, 64)
    assert cl and list(idx) == list(range(10))


def test_cosine_hand_values(oracle):  # attention_test.cpp:249-266
    v, deg = oracle.cosine_similarity([1.0, 0.0], [1.0, 1.0])
    assert abs(v - 0.70710678118654752) <= 1e-12 * 0.70710678118654752 and not deg
    assert oracle.cosine_similarity([1.0, 0.0], [-1.0, 0.0])[0] == -1.0
    assert oracle.cosine_similarity([1.0, 0.0], [0.0, 0.0]) == (0.0, True)


# ----------------------------------------------------------- retrieval_test.cpp

def test_sign_bits_follow_projection(oracle):  # retrieval_test.cpp:55-67
    rng = np.random.default_rng(2)
    k = rng.standard_normal((32, 16))
    proj, bits = oracle.encode_sign_hash(k, 128, 99)
    assert proj.shape == (128, 16)
    for row in range(32):
        for b in range(128):
            dot = 0.0
            for c in range(16):
                dot += proj[b, c] * k[row, c]
            assert bool((int(bits[row, b // 64]) >> (b % 64)) & 1) == (dot >= 0.0)


def test_sign_hash_seed_determinism(oracle):  # retrieval_test.cpp:69-77
    k = np.random.default_rng(3).standard_normal((40, 12))
    a = oracle.encode_sign_hash(k, 256, 5)[1]
    b = oracle.encode_sign_hash(k, 256, 5)[1]
    c = oracle.encode_sign_hash(k, 256, 6)[1]
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_retrieval_scale_invariance(oracle):  # retrieval_test.cpp:112-129
    rng = np.random.default_rng(6)
    k, q = rng.standard_normal((64, 16)), rng.standard_normal(16)
    for variant in (0, 1):
        a = oracle.retrieve_scored(q, k, 9, variant=variant, seed=17)[0]
        b = oracle.retrieve_scored(q * 3.7, k, 9, variant=variant, seed=17)[0]
        assert np.array_equal(a, b)
    ks = k.copy()
    ks[20] *= 5.0
    assert np.array_equal(oracle.encode_sign_hash(k, 256, 17)[1], oracle.encode_sign_hash(ks, 256, 17)[1])


def test_sign_hash_recovers_top1(oracle):  # retrieval_test.cpp:131-154 (>= 950/1000)
    rng = np.random.default_rng(1234)
    rec = 0
    for _ in range(200):
        k = rng.standard_normal((64, 16))
        k /= np.linalg.norm(k, axis=1, keepdims=True)
        target = rng.integers(64)
        q = k[target] + 0.1 * rng.standard_normal(16)
        want = oracle.topk_select_exact(q, k, 1)
        got = oracle.retrieve_scored(q, k, 1, variant=1, seed=555)[0]
        rec += int(np.array_equal(want, got))
    assert rec >= 190


def test_retrieval_argument_validation(oracle):  # retrieval_test.cpp:172-182
    k = np.zeros((4, 8))
    for kk in (5, 0):
        with pytest.raises(OracleError) as e:
            oracle.retrieve_scored(np.ones(8), k, kk)
        assert e.value.code == 2
    for bits in (0, 13):
        with pytest.raises(OracleError) as e:
            oracle.encode_sign_hash(k, bits, 1)
        assert e.value.code == 2


# ---------------------------------------------------- similarity_cache_test.cpp

def test_aggregate_hand_values(oracle):  # similarity_cache_test.cpp:44-54, :70-74
    assert abs(oracle.aggregate_similarity([0.5, 1.0], [1.0, 1.0]) - 2.0 / 3.0) < 1e-12
    assert abs(oracle.aggregate_similarity([0.5, 1.0], [0.9, 0.1]) - 1.0 / 1.9) < 1e-12
    assert abs(oracle.aggregate_similarity([0.5, 1.0], [0.0, 0.0]) - 2.0 / 3.0) < 1e-12


def test_aggregate_identity(oracle):  # similarity_cache_test.cpp:32-42
    rng = np.random.default_rng(11)
    for _ in range(200):
        m = 1 + rng.integers(8)
        w = rng.uniform(0.001, 1.0, m)
        assert abs(oracle.aggregate_similarity([0.9] * m, w) - 0.9) < 1e-12


def test_aggregate_validation(oracle):  # similarity_cache_test.cpp:76-85
    for sims, w in (([0.5, 1.0], [1.0, -0.5]), ([0.5, 0.0], [1.0, 1.0])):
        with pytest.raises(OracleError) as e:
            oracle.aggregate_similarity(sims, w)
        assert e.value.code == 2


def test_lookup_invalid_label_then_hit(oracle):  # similarity_cache_test.cpp:87-101
    q = np.array([[1.0, 0, 0, 0], [1.0, 0, 0, 0]])
    hit, agg, sims, reason, labels, valid = oracle.lookup(np.zeros((2, 4)), [0, 0], q, [1, 1], 0.5)
    assert not hit and reason == 1 and valid[0] == 1
    hit, agg, *_ = oracle.lookup(labels, valid, q, [1, 1], 0.5)
    assert hit and abs(agg - 1.0) < 1e-12


def test_lookup_non_positive_forces_miss(oracle):  # similarity_cache_test.cpp:103-116
    q = np.array([[1.0, 0, 0, 0], [1.0, 0, 0, 0]])
    lab = q.copy()
    lab[1, 0] = -1.0
    hit, _, _, reason, labels, _ = oracle.lookup(lab, [1, 1], q, [1, 1], -1.0)
    assert not hit and reason == 2 and np.array_equal(labels[1], q[1])


def test_lookup_below_threshold(oracle):  # similarity_cache_test.cpp:118-130
    hit, agg, _, reason, _, _ = oracle.lookup([[1.0, 0, 0, 0]], [1], [[0.9, 0.1, 0, 0]], [1.0], 0.9999)
    assert not hit and reason == 3 and 0.9 < agg < 0.9999


def test_merge_examples(oracle):  # similarity_cache_test.cpp:278-294
    props = [[(4, 9.0), (1, 5.0), (7, 2.0)], [(1, 8.0), (2, 6.0), (9, 1.0)]]
    assert list(oracle.merge_group_topk(props, 3)) == [1, 2, 4]
    assert list(oracle.merge_group_topk(props, 5)) == [1, 2, 4, 7, 9]
    assert list(oracle.merge_group_topk([[(8, 3.0), (2, 3.0)], [(5, 3.0)]], 2)) == [2, 5]
    for k in (0, 2):
        with pytest.raises(OracleError):
            oracle.merge_group_topk([[(1, 2.0)]], k)


def test_cache_bytes(oracle):  # similarity_cache_test.cpp:264-276
    assert oracle.cache_bytes(1, 1000, 0, 0, 0, 128, 2) == 512000
    one = oracle.cache_bytes(1, 100, 68, 4, 8, 64, 2)
    two = oracle.cache_bytes(2, 100, 68, 4, 8, 64, 2)
    lab = oracle.cache_bytes(0, 100, 68, 4, 8, 64, 2)
    assert lab == 4 * 8 * 64 * 2 and two - one == one - lab


# -------------------------------------------------------- head_profile_test.cpp

def test_threshold_known_answer(oracle):  # head_profile_test.cpp:47-51
    assert oracle.compute_threshold(0.5, 0.8, 3.0) == pytest.approx(-0.95164126255001177, abs=1e-15)
    assert oracle.compute_threshold(1.0, 0.8, 3.0) == pytest.approx(0.8, abs=1e-15)
    assert oracle.compute_threshold(0.0, 0.8, 3.0) == pytest.approx(-1.0, abs=1e-15)


def test_plan_partition_layer0_and_np(oracle):  # head_profile_test.cpp:202-212 (N_p)
    diff = np.array([[0.5, -0.1, 0.3, 0.2], [0.4, 0.1, -0.2, 0.3], [-1, -1, 0.9, 0.8]])
    pers, n_p, dropped = oracle.plan_partition(diff, t_comp_s=1e-4, pcie_bw=2e10, mem_head_bytes=2e5)
    assert n_p == 10
    assert pers[0].all() and not pers[1:].any() and dropped == 0
    pers, n_p, _ = oracle.plan_partition(diff, t_comp_s=1e-5, pcie_bw=2e10, mem_head_bytes=2e5)
    assert n_p == 1
    assert list(pers[1]) == [True, False, False, True] and list(pers[2]) == [False, False, True, False]
