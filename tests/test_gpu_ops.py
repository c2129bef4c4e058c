"""Op-level parity of the CUDA kernels behind the C-ABI against the CPU oracle
(and, for the known-answer cases, the reference's own golden vectors).
Bit-exact for indices / bits / decisions / rows; attention within 1e-12
relative for f64 storage and the north-star tolerances otherwise."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2511_14510_b200 import _lib  # noqa: E402
from paper_2511_14510_b200.workload import bf16_bits_to_f32, f32_to_bf16_bits  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


_KEEP = []


def dev(a, dtype=None):
    """Device copy of a numpy array. Kept alive for the test's duration so
    `dev(x).data_ptr()` can be passed inline to the C-ABI."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    t = t.to(DEV) if dtype is None else t.to(DEV, dtype)
    _KEEP.append(t)
    return t


@pytest.fixture(autouse=True)
def _release_kept():
    yield
    torch.cuda.synchronize()
    _KEEP.clear()


def group_topk(lib, q, keys, k, retriever, dtype=_lib.DTYPE_F64, seed=0, bits=256):
    q = np.atleast_2d(q)
    m, d = q.shape
    n = keys.shape[0]
    qd = dev(q.astype(np.float64))
    kd = dev(keys)
    codes = None
    if retriever == _lib.RETRIEVER_SIGN_HASH:
        codes = torch.empty((n, (bits + 63) // 64), dtype=torch.int64, device=DEV)
        _lib.check(lib.clo_encode_sign_hash(kd.data_ptr(), dtype, n, d, bits, seed, codes.data_ptr(), None))
    out = torch.empty(k, dtype=torch.int32, device=DEV)
    sc = torch.empty(k, dtype=torch.float64, device=DEV)
    _lib.check(lib.clo_group_topk(qd.data_ptr(), m, d, retriever, kd.data_ptr(), dtype,
                                  None if codes is None else codes.data_ptr(), bits, seed, n, k,
                                  out.data_ptr(), sc.data_ptr(), None))
    return out.cpu().numpy(), sc.cpu().numpy(), codes


@pytest.mark.parametrize("retriever", [_lib.RETRIEVER_EXACT, _lib.RETRIEVER_SIGN_HASH])
def test_retrieve_scored_matches_oracle(clo, oracle, retriever):
    rng = np.random.default_rng(retriever)
    for trial in range(20):
        n, d = int(rng.integers(50, 3000)), int(rng.choice([8, 16, 32, 128]))
        k = int(rng.integers(1, min(n, 600)))
        keys = rng.standard_normal((n, d))
        if trial % 4 == 0:  # ties: repeated rows, coarse values
            keys = np.round(keys)
            keys[n // 3:] = keys[: n - n // 3]
        q = rng.standard_normal(d)
        idx, sc, _ = group_topk(clo, q, keys, k, retriever, seed=trial)
        want_idx, want_sc = oracle.retrieve_scored(q, keys, k, variant=retriever, seed=trial)
        np.testing.assert_array_equal(idx, want_idx)
        np.testing.assert_array_equal(sc, want_sc)


@pytest.mark.parametrize("retriever", [_lib.RETRIEVER_EXACT, _lib.RETRIEVER_SIGN_HASH])
def test_fused_group_topk_equals_merge_of_per_head_topk(clo, oracle, retriever):
    # engine.cpp:211-223: m retrieve_scored + merge_group_topk == one top-k over max_j
    rng = np.random.default_rng(10 + retriever)
    for trial in range(20):
        n, d, m = int(rng.integers(100, 5000)), 32, int(rng.integers(2, 6))
        k = int(rng.integers(1, 300))
        keys = rng.standard_normal((n, d))
        if trial % 3 == 0:
            keys = np.round(keys * 2) / 2
        qs = rng.standard_normal((m, d))
        props = []
        for j in range(m):
            i, s = oracle.retrieve_scored(qs[j], keys, k, variant=retriever, seed=trial)
            props.append(list(zip(map(int, i), map(float, s))))
        want = oracle.merge_group_topk(props, k)
        got, _, _ = group_topk(clo, qs, keys, k, retriever, seed=trial)
        np.testing.assert_array_equal(got, want)


def test_encode_bits_match_oracle(clo, oracle):
    rng = np.random.default_rng(2)
    for bits in (8, 64, 128, 256, 512):
        keys = rng.standard_normal((700, 24))
        kd = dev(keys)
        codes = torch.empty((700, (bits + 63) // 64), dtype=torch.int64, device=DEV)
        _lib.check(clo.clo_encode_sign_hash(kd.data_ptr(), _lib.DTYPE_F64, 700, 24, bits, 99,
                                            codes.data_ptr(), None))
        _, want = oracle.encode_sign_hash(keys, bits, 99)
        np.testing.assert_array_equal(codes.cpu().numpy().view(np.uint64), want)


def test_projection_matches_libstdcxx_stream(clo, oracle):
    p = np.zeros((256, 128))
    _lib.check(clo.clo_sign_hash_projection(256, 128, 12345, p.ctypes.data))
    np.testing.assert_array_equal(p.ravel(), oracle.fill_normal(12345, 256 * 128))


def test_topk_select_golden_ties(clo):
    # attention_test.cpp:119-131
    k = np.zeros((5, 2))
    k[:, 0] = [0.5, 1.0, 2.0, 1.0, 0.5]
    for kk, want in ((2, [1, 2]), (3, [1, 2, 3]), (4, [0, 1, 2, 3])):
        got, _, _ = group_topk(clo, [1.0, 0.0], k, kk, _lib.RETRIEVER_EXACT)
        assert list(got) == want


def test_topk_select_argument_errors(clo):
    with pytest.raises(_lib.ArgumentError):
        group_topk(clo, [1.0, 0.0], np.zeros((4, 2)), 5, _lib.RETRIEVER_EXACT)


def test_negative_zero_ties_with_positive_zero(clo, oracle):
    keys = np.array([[1.0], [-1.0], [0.0], [1.0]])
    q = np.array([0.0])  # every score is +-0.0: all tie, lower index wins
    got, _, _ = group_topk(clo, q, keys, 2, _lib.RETRIEVER_EXACT)
    assert list(got) == list(oracle.retrieve_scored(q, keys, 2)[0]) == [0, 1]


def test_merge_group_topk_golden(clo):
    # similarity_cache_test.cpp:278-294
    def merge(props, k):
        sizes = np.array([len(p) for p in props], np.int32)
        idx = dev(np.array([i for p in props for i, _ in p], np.int32))
        sc = dev(np.array([s for p in props for _, s in p], np.float64))
        out = torch.empty(k, dtype=torch.int32, device=DEV)
        _lib.check(clo.clo_merge_group_topk(sizes.ctypes.data, len(props), idx.data_ptr(), sc.data_ptr(), k,
                                            out.data_ptr(), None))
        return list(out.cpu().numpy())
    props = [[(4, 9.0), (1, 5.0), (7, 2.0)], [(1, 8.0), (2, 6.0), (9, 1.0)]]
    assert merge(props, 3) == [1, 2, 4]
    assert merge(props, 5) == [1, 2, 4, 7, 9]
    assert merge([[(8, 3.0), (2, 3.0)], [(5, 3.0)]], 2) == [2, 5]


def test_lookup_matches_oracle(clo, oracle):
    rng = np.random.default_rng(4)
    H, m, d = 64, 4, 128
    labels = rng.standard_normal((H, m, d))
    valid = (rng.random((H, m)) > 0.05).astype(np.int32)
    queries = labels + rng.uniform(0.1, 2.0, (H, 1, 1)) * rng.standard_normal((H, m, d))
    weights = rng.uniform(0, 1, (H, m))
    weights[3] = 0.0  # all-zero weights fall back to uniform
    tau = rng.uniform(-0.5, 0.99, H)
    dl, dv = dev(labels), dev(valid)
    hit = torch.empty(H, dtype=torch.int32, device=DEV)
    agg = torch.empty(H, dtype=torch.float64, device=DEV)
    sims = torch.empty((H, m), dtype=torch.float64, device=DEV)
    reason = torch.empty(H, dtype=torch.int32, device=DEV)
    _lib.check(clo.clo_lookup(H, m, d, dl.data_ptr(), dv.data_ptr(), dev(queries).data_ptr(),
                              dev(weights).data_ptr(), dev(tau).data_ptr(), hit.data_ptr(), agg.data_ptr(),
                              sims.data_ptr(), reason.data_ptr(), None))
    for h in range(H):
        w = oracle.lookup(labels[h], valid[h], queries[h], weights[h], tau[h])
        assert bool(hit[h]) == w[0] and agg[h].item() == w[1] and reason[h].item() == w[3]
        np.testing.assert_array_equal(sims[h].cpu().numpy(), w[2])
        np.testing.assert_array_equal(dl[h].cpu().numpy(), w[4])
        np.testing.assert_array_equal(dv[h].cpu().numpy(), w[5])


def test_lookup_golden(clo):
    # similarity_cache_test.cpp:87-101: invalid label -> miss, refresh, then hit at 1.0
    d = 4
    lab = torch.zeros((1, 2, d), dtype=torch.float64, device=DEV)
    val = torch.zeros((1, 2), dtype=torch.int32, device=DEV)
    q = dev(np.array([[[1.0, 0, 0, 0], [1.0, 0, 0, 0]]]))
    w = dev(np.ones((1, 2)))
    tau = dev(np.array([0.5]))
    outs = [torch.empty(1, dtype=torch.int32, device=DEV), torch.empty(1, dtype=torch.float64, device=DEV),
            torch.empty((1, 2), dtype=torch.float64, device=DEV), torch.empty(1, dtype=torch.int32, device=DEV)]

    def call():
        _lib.check(clo.clo_lookup(1, 2, d, lab.data_ptr(), val.data_ptr(), q.data_ptr(), w.data_ptr(),
                                  tau.data_ptr(), *[o.data_ptr() for o in outs], None))
        return outs[0].item(), outs[1].item(), outs[3].item()
    assert call() == (0, 0.0, 1)
    hit, agg, reason = call()
    assert hit == 1 and abs(agg - 1.0) < 1e-12 and reason == 0


def test_aggregate_and_cosine_golden(clo):
    sims = dev(np.array([[0.5, 1.0], [0.5, 1.0], [0.5, 1.0]]))
    w = dev(np.array([[1.0, 1.0], [0.9, 0.1], [0.0, 0.0]]))
    out = torch.empty(3, dtype=torch.float64, device=DEV)
    _lib.check(clo.clo_aggregate_similarity(3, 2, sims.data_ptr(), w.data_ptr(), out.data_ptr(), None))
    np.testing.assert_allclose(out.cpu().numpy(), [2 / 3, 1 / 1.9, 2 / 3], rtol=1e-12)
    with pytest.raises(_lib.ArgumentError):
        bad = dev(np.array([[0.5, 0.0]]))
        _lib.check(clo.clo_aggregate_similarity(1, 2, bad.data_ptr(), w.data_ptr(), out.data_ptr(), None))
    a = dev(np.array([[1.0, 0.0], [1.0, 0.0], [1.0, 0.0]]))
    b = dev(np.array([[1.0, 1.0], [-1.0, 0.0], [0.0, 0.0]]))
    val = torch.empty(3, dtype=torch.float64, device=DEV)
    deg = torch.empty(3, dtype=torch.int32, device=DEV)
    _lib.check(clo.clo_cosine_similarity(3, 2, a.data_ptr(), b.data_ptr(), val.data_ptr(), deg.data_ptr(), None))
    v = val.cpu().numpy()
    assert abs(v[0] - 0.70710678118654752) < 1e-15 and v[1] == -1.0 and v[2] == 0.0
    assert list(deg.cpu().numpy()) == [0, 0, 1]


@pytest.mark.parametrize("kv_dtype", ["bf16", "f32"])
def test_zero_copy_gather_is_bit_exact(clo, kv_dtype):
    rng = np.random.default_rng(1)
    n, d, k = 50000, 128, 2048
    x = rng.standard_normal((n, d)).astype(np.float32)
    host = f32_to_bf16_bits(x) if kv_dtype == "bf16" else x
    p = C.c_void_p()
    _lib.check(clo.clo_host_alloc(host.nbytes, C.byref(p)))
    try:
        buf = np.frombuffer((C.c_char * host.nbytes).from_address(p.value), dtype=host.dtype).reshape(host.shape)
        buf[:] = host
        idx = np.sort(rng.choice(n, k, replace=False)).astype(np.int32)
        dst = torch.empty((k, d), dtype=torch.int16 if kv_dtype == "bf16" else torch.float32, device=DEV)
        dt = _lib.DTYPE_BF16 if kv_dtype == "bf16" else _lib.DTYPE_F32
        _lib.check(clo.clo_gather_rows(p.value, dt, d, n, dev(idx).data_ptr(), k, dst.data_ptr(), None))
        got = dst.cpu().numpy()
        want = host[idx]
        np.testing.assert_array_equal(got.view(want.dtype), want)
        bad = dev(np.array([n], np.int32))
        with pytest.raises(_lib.IndexError_):
            _lib.check(clo.clo_gather_rows(p.value, dt, d, n, bad.data_ptr(), 1, dst.data_ptr(), None))
    finally:
        clo.clo_host_free(p.value)


@pytest.mark.parametrize("kv_dtype", ["f64", "f32", "bf16"])
def test_topk_attention_matches_oracle(clo, oracle, kv_dtype):
    rng = np.random.default_rng(7)
    n, d, m = 3000, 128, 4
    kf, vf = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    if kv_dtype == "bf16":
        kb, vb = f32_to_bf16_bits(kf.astype(np.float32)), f32_to_bf16_bits(vf.astype(np.float32))
        kw, vw = bf16_bits_to_f32(kb).astype(np.float64), bf16_bits_to_f32(vb).astype(np.float64)
        kd, vd, dt, tol = dev(kb.view(np.int16)), dev(vb.view(np.int16)), _lib.DTYPE_BF16, 2e-2
    elif kv_dtype == "f32":
        kf32, vf32 = kf.astype(np.float32), vf.astype(np.float32)
        kw, vw = kf32.astype(np.float64), vf32.astype(np.float64)
        kd, vd, dt, tol = dev(kf32), dev(vf32), _lib.DTYPE_F32, 1e-3
    else:
        kw, vw = kf, vf
        kd, vd, dt, tol = dev(kf), dev(vf), _lib.DTYPE_F64, 1e-12
    q = rng.standard_normal((m, d))
    idx = np.sort(rng.choice(n, 2116, replace=False)).astype(np.int32)
    out = torch.empty((m, d), dtype=torch.float64, device=DEV)
    _lib.check(clo.clo_topk_attention(dev(q).data_ptr(), m, kd.data_ptr(), vd.data_ptr(), dt, n, d,
                                      dev(idx).data_ptr(), len(idx), out.data_ptr(), None))
    got = out.cpu().numpy()
    for j in range(m):
        want = oracle.topk_attention(q[j], kw, vw, idx)
        assert np.linalg.norm(got[j] - want) / np.linalg.norm(want) <= tol


def test_topk_attention_golden_and_errors(clo):
    # attention_test.cpp:29-38 single token; :170-179 bad index sets; :83-92 NaN
    k = dev(np.array([[2.0, 0, 0]]))
    v = dev(np.array([[5.0, -1.0, 0.25]]))
    q = dev(np.array([[1.0, 0, 0]]))
    out = torch.empty((1, 3), dtype=torch.float64, device=DEV)
    _lib.check(clo.clo_topk_attention(q.data_ptr(), 1, k.data_ptr(), v.data_ptr(), _lib.DTYPE_F64, 1, 3,
                                      dev(np.array([0], np.int32)).data_ptr(), 1, out.data_ptr(), None))
    assert list(out.cpu().numpy()[0]) == [5.0, -1.0, 0.25]
    K4, V4 = dev(np.zeros((4, 2))), dev(np.zeros((4, 2)))
    q2 = dev(np.array([[1.0, 0.0]]))
    o2 = torch.empty((1, 2), dtype=torch.float64, device=DEV)
    for idx, exc in (([4], _lib.IndexError_), ([1, 1], _lib.ArgumentError)):
        with pytest.raises(exc):
            _lib.check(clo.clo_topk_attention(q2.data_ptr(), 1, K4.data_ptr(), V4.data_ptr(), _lib.DTYPE_F64, 4, 2,
                                              dev(np.array(idx, np.int32)).data_ptr(), len(idx), o2.data_ptr(),
                                              None))
    Kn = np.zeros((4, 2))
    Kn[0, 0] = np.nan
    with pytest.raises(_lib.NumericError):
        _lib.check(clo.clo_topk_attention(q2.data_ptr(), 1, dev(Kn).data_ptr(), V4.data_ptr(), _lib.DTYPE_F64, 4,
                                          2, dev(np.array([1], np.int32)).data_ptr(), 1, o2.data_ptr(), None))


@pytest.mark.parametrize("huge", [0, 1])
def test_numa_bound_host_store_gathers_bit_exact(clo, huge):
    """clo_host_alloc_numa: the store is bound to the GPU's NUMA node (node 0
    when the host reports none) and pinned; zero-copy gathers from it are
    bit-exact with both copy engines."""
    from paper_2511_14510_b200.engine import device_numa_node
    node = device_numa_node(0)
    assert node >= -1
    n, d = 5000, 128
    nbytes = n * d * 2
    p = C.c_void_p()
    _lib.check(clo.clo_host_alloc_numa(nbytes, huge, max(node, 0), C.byref(p)))
    try:
        host = np.frombuffer((C.c_char * nbytes).from_address(p.value), dtype=np.uint16).reshape(n, d)
        host[:] = np.random.default_rng(3).integers(0, 65535, host.shape, dtype=np.uint16)
        idx = np.sort(np.random.default_rng(4).choice(n, 777, replace=False)).astype(np.int32)
        err = torch.zeros(1, dtype=torch.int32, device=DEV)
        for engine in (0, 1):
            out = torch.empty((len(idx), d), dtype=torch.int16, device=DEV)
            _lib.check(clo.clo_gather_rows_ex(p.value, _lib.DTYPE_BF16, d, n, dev(idx).data_ptr(), len(idx),
                                              out.data_ptr(), engine, 0, err.data_ptr(), None))
            torch.cuda.synchronize()
            assert int(err.item()) == 0
            np.testing.assert_array_equal(out.cpu().numpy().view(np.uint16), host[idx])
    finally:
        _lib.check(clo.clo_host_free(p.value))
