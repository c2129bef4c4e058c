"""Parity at BASELINE.json's full sizes (n = 131072 keys, d = 128, k = 2048,
m = 4) through size-independent checks the oracle can afford:
  * sign bits of sampled rows equal the oracle's (the bits depend only on the
    row and the seeded projection);
  * the fused group top-k equals an independent numpy top-k over
    S(i) = max_j (256 - popcount(q_j ^ code_i)) with (S desc, i asc);
  * the exact retriever equals the oracle's retrieve_scored + merge;
  * one full-size engine step: gathered rows are the host rows bit for bit
    and attention matches an fp64 recomputation over union(entry, window)."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2511_14510_b200 import _lib  # noqa: E402
from paper_2511_14510_b200.workload import bf16_bits_to_f32, f32_to_bf16_bits  # noqa: E402

pytestmark = pytest.mark.gpu
N, D, K, M, BITS = 131072, 128, 2048, 4, 256


def _keys(seed):
    rng = np.random.default_rng(seed)
    kb = f32_to_bf16_bits(rng.standard_normal((N, D), np.float32))
    return kb, bf16_bits_to_f32(kb).astype(np.float64), rng


def test_fullsize_sign_hash_bits_and_topk(clo, oracle):
    kb, kw, rng = _keys(1)
    dk = torch.from_numpy(kb.view(np.int16)).cuda()
    codes = torch.empty((N, 4), dtype=torch.int64, device="cuda")
    seed = 0x5EED
    _lib.check(clo.clo_encode_sign_hash(dk.data_ptr(), _lib.DTYPE_BF16, N, D, BITS, seed, codes.data_ptr(), None))
    cg = codes.cpu().numpy().view(np.uint64)
    sample = rng.choice(N, 1500, replace=False)
    proj, want_bits = oracle.encode_sign_hash(kw[sample], BITS, seed)
    np.testing.assert_array_equal(cg[sample], want_bits)
    q = rng.standard_normal((M, D))
    qd = torch.from_numpy(q).cuda()
    out = torch.empty(K, dtype=torch.int32, device="cuda")
    sc = torch.empty(K, dtype=torch.float64, device="cuda")
    _lib.check(clo.clo_group_topk(qd.data_ptr(), M, D, _lib.RETRIEVER_SIGN_HASH, dk.data_ptr(), _lib.DTYPE_BF16,
                                  codes.data_ptr(), BITS, seed, N, K, out.data_ptr(), sc.data_ptr(), None))
    _, qbits = oracle.encode_sign_hash(q, BITS, seed)  # query bits: same projection, same arithmetic
    S = np.zeros(N, np.int64)
    for j in range(M):
        dist = np.bitwise_count(cg ^ qbits[j][None, :]).sum(axis=1).astype(np.int64)
        S = np.maximum(S, BITS - dist)
    order = np.lexsort((np.arange(N), -S))[:K]
    np.testing.assert_array_equal(out.cpu().numpy(), np.sort(order))
    np.testing.assert_array_equal(sc.cpu().numpy(), S[np.sort(order)].astype(np.float64))


def test_fullsize_exact_group_topk(clo, oracle):
    kb, kw, rng = _keys(2)
    q = rng.standard_normal((M, D))
    dk = torch.from_numpy(kb.view(np.int16)).cuda()
    qd = torch.from_numpy(q).cuda()
    out = torch.empty(K, dtype=torch.int32, device="cuda")
    _lib.check(clo.clo_group_topk(qd.data_ptr(), M, D, _lib.RETRIEVER_EXACT, dk.data_ptr(), _lib.DTYPE_BF16,
                                  None, 0, 0, N, K, out.data_ptr(), None, None))
    props = []
    for j in range(M):
        i, s = oracle.retrieve_scored(q[j], kw, K)
        props.append(list(zip(map(int, i), map(float, s))))
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.merge_group_topk(props, K))


def test_fullsize_engine_step_rows_and_attention():
    from paper_2511_14510_b200 import (DecodeEngine, EngineConfig, ModeFlags, ModelShape,
                                       layer0_only_plan, uniform_profiles)
    from paper_2511_14510_b200.workload import Shape, SyntheticWorkload
    L, HQ, H = 2, 32, 8
    wl = SyntheticWorkload(Shape(L, HQ, H, D), 1, N, 2, kv_dtype="bf16", sigma_step=0.05, seed=3,
                           alias_layers=True)
    cfg = EngineConfig(shape=ModelShape(L, HQ, H, D, 2), k=K, retriever="sign_hash", batch=1,
                       kv_dtype="bf16", collect_outputs=True, mode=ModeFlags(always_miss=True))
    eng = DecodeEngine(cfg, uniform_profiles(cfg.shape, 0.5), layer0_only_plan(cfg.shape), wl)
    eng.run()
    out = eng.collected_outputs()[-1][0]  # [L][hq][d] of the last step
    hk = bf16_bits_to_f32(eng.hkv.k[0, 0]).astype(np.float64)  # [H][nmax][d] host store
    hv = bf16_bits_to_f32(eng.hkv.v[0, 0]).astype(np.float64)
    n_after = N + 2
    window = list(range(4)) + list(range(n_after - 64, n_after))
    m = HQ // H
    worst = 0.0
    for g in range(H):
        st = eng.head(1, g)
        idx = st["entry_indices"]
        kr, vr = eng.entry_rows(1, g)
        np.testing.assert_array_equal(kr, eng.hkv.k[0, 0, g][idx])  # gathered rows, bit for bit
        np.testing.assert_array_equal(vr, eng.hkv.v[0, 0, g][idx])
        attend = np.union1d(idx, window)
        for j in range(m):
            q = wl.true_q[2, 0, 1, g * m + j].astype(np.float64)
            s = hk[g][attend] @ q / np.sqrt(D)
            w = np.exp(s - s.max())
            want = (w / w.sum()) @ hv[g][attend]
            got = out[1, g * m + j]
            worst = max(worst, float(np.linalg.norm(got - want) / np.linalg.norm(want)))
    assert worst < 1e-4, worst
