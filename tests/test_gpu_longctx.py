"""Parity at the long-context BASELINE configs: configs[2] (Qwen2.5-14B-1M
shape, 40q/8kv so m = 5, 512K context, plan_partition persistent heads) and
configs[3] (1M context, KV-head shards).

Selection at these sizes runs the threshold kernel's long-item branch
(select.cu: more than 64 chunks of 4096 keys per item, warp-parallel chunk
sums) and spreads the tie quota over hundreds of chunks. Checked here, with
size-independent references the CPU affords:
  * sign bits of sampled rows vs the C oracle (encode, retrieval.cpp:14-25);
  * the fused group top-k vs an independent numpy top-k over
    S(i) = max_j (256 - popcount(q_j ^ code_i)) ordered (S desc, i asc) —
    select_topk (retrieval.cpp:33-46) + retrieve_scored (:90-125) + the merge
    (similarity_cache.cpp:180-201), DESIGN.md §3;
  * a tie-heavy key set (16 distinct rows tiled over n) where the k-th score
    level holds tens of thousands of ties resolved by index across >64 chunks;
  * engine steps at 512K (m = 5, persistent heads beyond layer 0 from
    plan_partition, head_profile.cpp:80-154; persistent serve path
    engine.cpp:269-274) and 1M (a KV-head shard): every entry equals the numpy
    top-k of its query over the n_pool = n_prompt + t - 1 rows, gathered rows
    equal the host rows bit for bit, and attention matches an fp64
    recomputation over union(entry, sink/recent window) within 1e-4."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2511_14510_b200 import _lib  # noqa: E402
from paper_2511_14510_b200.workload import bf16_bits_to_f32  # noqa: E402

pytestmark = pytest.mark.gpu
D, K, BITS = 128, 2048, 256


def _bf16_rows(gen, n, device="cuda"):
    return torch.randn((n, D), generator=gen, device=device, dtype=torch.float32).to(torch.bfloat16)


def _encode(clo, keys_bf16, seed):
    n = keys_bf16.shape[0]
    codes = torch.empty((n, BITS // 64), dtype=torch.int64, device="cuda")
    _lib.check(clo.clo_encode_sign_hash(keys_bf16.data_ptr(), _lib.DTYPE_BF16, n, D, BITS, seed,
                                        codes.data_ptr(), None))
    return codes


def _numpy_topk(codes_u64, qbits, k):
    """(S desc, index asc) top-k over S(i) = max_j (bits - popcount(q_j ^ code_i)), ascending."""
    S = np.zeros(codes_u64.shape[0], np.int64)
    for j in range(qbits.shape[0]):
        dist = np.bitwise_count(codes_u64 ^ qbits[j][None, :]).sum(axis=1).astype(np.int64)
        S = np.maximum(S, BITS - dist)
    order = np.lexsort((np.arange(S.shape[0]), -S))[:k]
    return np.sort(order), S


def _group_topk(clo, q, keys, codes, seed, k=K):
    n = keys.shape[0]
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float64)).cuda()
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    sc = torch.empty(k, dtype=torch.float64, device="cuda")
    _lib.check(clo.clo_group_topk(qd.data_ptr(), q.shape[0], D, _lib.RETRIEVER_SIGN_HASH, keys.data_ptr(),
                                  _lib.DTYPE_BF16, codes.data_ptr(), BITS, seed, n, k, out.data_ptr(),
                                  sc.data_ptr(), None))
    return out.cpu().numpy(), sc.cpu().numpy()


@pytest.mark.parametrize("n,m", [(524288, 5), (524288, 4), (1048576, 4), (1048576, 5)])
def test_longctx_group_topk(clo, oracle, n, m):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(n + m)
    keys = _bf16_rows(gen, n)
    seed = oracle.mix_seed3(1, 7, m)
    codes = _encode(clo, keys, seed)
    cg = codes.cpu().numpy().view(np.uint64)
    rng = np.random.default_rng(n + m)
    sample = rng.choice(n, 800, replace=False)
    kw = bf16_bits_to_f32(keys[torch.from_numpy(sample).cuda()].view(torch.int16).cpu().numpy().view(np.uint16))
    _, want_bits = oracle.encode_sign_hash(kw.astype(np.float64), BITS, seed)
    np.testing.assert_array_equal(cg[sample], want_bits)
    q = rng.standard_normal((m, D))
    got, got_s = _group_topk(clo, q, keys, codes, seed)
    _, qbits = oracle.encode_sign_hash(q, BITS, seed)
    want, S = _numpy_topk(cg, qbits, K)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got_s, S[want].astype(np.float64))


@pytest.mark.parametrize("n,m", [(524288, 5), (1048576, 4)])
def test_longctx_tie_heavy_threshold(clo, oracle, n, m):
    """16 distinct key rows tiled over n: S takes at most 16 values, so the k-th
    level holds ~n/16 ties and the tie quota (first `need` ties in index order)
    is spread over every one of the n/4096 > 64 chunks."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(99 + n)
    base = _bf16_rows(gen, 16)
    perm = torch.randint(0, 16, (n,), generator=gen, device="cuda")
    keys = base[perm].contiguous()
    seed = oracle.mix_seed3(3, 1, 4)
    codes = _encode(clo, keys, seed)
    cg = codes.cpu().numpy().view(np.uint64)
    assert len(np.unique(cg, axis=0)) <= 16
    rng = np.random.default_rng(5)
    for trial in range(3):
        q = rng.standard_normal((m, D))
        _, qbits = oracle.encode_sign_hash(q, BITS, seed)
        want, S = _numpy_topk(cg, qbits, K)
        T = np.sort(S)[::-1][K - 1]
        assert (S == T).sum() > 64 * 4, "the k-th level must hold ties across many chunks"
        got, _ = _group_topk(clo, q, keys, codes, seed)
        np.testing.assert_array_equal(got, want, err_msg=f"trial {trial}")


def _run_engine(oracle, *, n, L, HQ, H, kv0, persistent, steps=2, batch=1, seed=11):
    """Bench-shaped engine (aliased interleaved host store, device-resident step
    inputs, always_miss so every offloaded head reselects with its approximate
    query every step). Returns what the checks need."""
    from paper_2511_14510_b200.engine import (DecodeEngine, EngineConfig, HostKV, ModeFlags, ModelShape,
                                              PartitionPlan, profiles_from_arrays)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    nmax = n + steps
    hkv = HostKV(batch, 1, H, nmax, D, "bf16", interleaved=True)
    kdev = torch.empty((batch, H, nmax, D), dtype=torch.bfloat16, device=dev)
    vdev = torch.empty_like(kdev)
    for b in range(batch):
        for h in range(H):
            kdev[b, h] = _bf16_rows(gen, nmax)
            vdev[b, h] = _bf16_rows(gen, nmax)
            torch.from_numpy(hkv.k[b, 0, h, :n].view(np.int16)).copy_(kdev[b, h, :n].view(torch.int16))
            torch.from_numpy(hkv.v[b, 0, h, :n].view(np.int16)).copy_(vdev[b, h, :n].view(torch.int16))
    m = HQ // H

    def norm(x):
        return x / x.norm(dim=-1, keepdim=True)
    q = norm(torch.randn((batch, L, HQ, D), generator=gen, device=dev))
    tq = torch.empty((steps + 1, batch, L, HQ, D), device=dev)
    aq = torch.empty_like(tq)
    for t in range(steps + 1):
        if t:
            q = norm(q + 0.05 * torch.randn(q.shape, generator=gen, device=dev))
        tq[t] = q
        aq[t] = norm(q + 0.01 * torch.randn(q.shape, generator=gen, device=dev))
    # layer-invariant new rows (aliased store): row n + t - 1 of the device copy
    nk = torch.stack([kdev[:, :, n + t] for t in range(steps)])[:, :, None].expand(steps, batch, L, H, D).contiguous()
    nv = torch.stack([vdev[:, :, n + t] for t in range(steps)])[:, :, None].expand(steps, batch, L, H, D).contiguous()
    out = torch.empty((batch, L, HQ, D), device=dev)
    rng = np.random.default_rng(seed)
    tau = np.full((L, H), 0.5)
    qimp = rng.uniform(0, 1, (L, H, m))

    class _Src:
        n_prompt, alias_layers = n, True
        prompt_k = prompt_v = None
    _Src.steps = steps
    cfg = EngineConfig(shape=ModelShape(L, HQ, H, D, 2), k=K, sink_tokens=4, recent_tokens=64,
                       retriever="sign_hash", hash_bits=BITS, retriever_seed=1, policy="similarity",
                       mode=ModeFlags(always_miss=True), batch=batch, kv_dtype="bf16", kv_head_offset=kv0,
                       collect_outputs=True)
    plan = PartitionPlan(layers=[[g for g in range(H) if persistent[l, g]] for l in range(L)])
    eng = DecodeEngine(cfg, profiles_from_arrays(tau, qimp), plan, _Src, host_kv=hkv)
    lib = _lib.load()
    _lib.check(lib.clo_prefill(eng.h, tq[0].data_ptr(), 0, None))
    for t in range(1, steps + 1):
        io = _lib.StepIO(tq[t].data_ptr(), aq[t].data_ptr(), nk[t - 1].data_ptr(), nv[t - 1].data_ptr(),
                         out.data_ptr(), 0)
        _lib.check(lib.clo_decode_step(eng.h, C.byref(io), None))
    eng.metrics()  # synchronise; raises deferred device errors
    return dict(eng=eng, hkv=hkv, kdev=kdev, vdev=vdev, tq=tq, aq=aq, out=out.cpu().numpy(), n=n, L=L, HQ=HQ,
                H=H, m=m, kv0=kv0, steps=steps, persistent=persistent, batch=batch)


def _check_engine(clo, oracle, r, layers):
    eng, n, steps, m = r["eng"], r["n"], r["steps"], r["m"]
    n_pool, n_after = n + steps - 1, n + steps
    window = np.union1d(np.arange(4), np.arange(n_after - 64, n_after))
    worst = 0.0
    checked = {"persistent": 0, "offloaded": 0}
    for b in range(r["batch"]):
        for l in layers:
            for g in range(r["H"]):
                pers = bool(r["persistent"][l, g])
                seed = oracle.mix_seed3(1, l, g + r["kv0"])
                keys = r["kdev"][b, g, :n_pool].contiguous()
                cg = _encode(clo, keys, seed).cpu().numpy().view(np.uint64)
                src = r["tq"] if pers else r["aq"]
                q = src[steps, b, l, g * m:(g + 1) * m].double().cpu().numpy()
                _, qbits = oracle.encode_sign_hash(q, BITS, seed)
                want, _ = _numpy_topk(cg, qbits, K)
                st = eng.head(l, g, seq=b)
                where = f"seq {b} layer {l} head {g} ({'persistent' if pers else 'offloaded'})"
                np.testing.assert_array_equal(st["entry_indices"], want, err_msg=where)
                checked["persistent" if pers else "offloaded"] += 1
                attend = np.union1d(want, window)
                at = torch.from_numpy(attend).cuda()

                def rows(x):
                    return bf16_bits_to_f32(x[b, g][at].view(torch.int16).cpu().numpy().view(np.uint16)).astype(np.float64)
                hk, hv = rows(r["kdev"]), rows(r["vdev"])
                if not pers:  # gathered entry rows = host rows, bit for bit
                    kr, vr = eng.entry_rows(l, g, seq=b)
                    np.testing.assert_array_equal(kr, r["hkv"].k[b, 0, g][want], err_msg=where)
                    np.testing.assert_array_equal(vr, r["hkv"].v[b, 0, g][want], err_msg=where)
                for j in range(m):
                    qq = r["tq"][steps, b, l, g * m + j].double().cpu().numpy()
                    s = hk @ qq / np.sqrt(D)
                    w = np.exp(s - s.max())
                    want_o = (w / w.sum()) @ hv
                    got = r["out"][b, l, g * m + j]
                    worst = max(worst, float(np.linalg.norm(got - want_o) / np.linalg.norm(want_o)))
    assert worst < 1e-4, worst
    return checked


def test_longctx_qwen_512k_engine_plan_partition(clo, oracle):
    """configs[2] shape: 40q/8kv (m = 5), 512K context, a plan_partition plan
    with persistent heads beyond layer 0 (n_p = floor(5e-5 * 5e10 / 1 MiB) = 2;
    layer 1 has 5 heads of positive difficulty, so its 3 hardest persist)."""
    L, HQ, H, n = 3, 40, 8, 524288
    diff = np.array([[0.1] * H,
                     [0.3, 0.5, -0.1, 0.2, 0.4, -0.2, 0.1, -0.3],
                     [-0.1] * H])
    pers = np.zeros((L, H), np.int32)
    n_p, nd = C.c_int(), C.c_int()
    lib = _lib.load()
    _lib.check(lib.clo_plan_partition(np.ascontiguousarray(diff).ctypes.data, L, H, 5e-5, 5.0e10,
                                      float(2 * K * D * 2), 0, 0, pers.ctypes.data, C.byref(n_p), C.byref(nd)))
    assert n_p.value == 2
    assert pers[0].all() and pers[1].tolist() == [1, 1, 0, 0, 1, 0, 0, 0] and not pers[2].any()
    r = _run_engine(oracle, n=n, L=L, HQ=HQ, H=H, kv0=0, persistent=pers)
    checked = _check_engine(clo, oracle, r, layers=[1, 2])
    assert checked == {"persistent": 3, "offloaded": 13}


def test_longctx_1m_kv_head_shard_engine(clo, oracle):
    """configs[3] shape, one KV-head shard of four (rank 1: KV heads 2-3, query
    heads 8-15), 1M context: seeds and profiles follow the global head index."""
    L, HQ, H, n = 2, 8, 2, 1048576
    pers = np.zeros((L, H), np.int32)
    pers[0] = 1
    r = _run_engine(oracle, n=n, L=L, HQ=HQ, H=H, kv0=2, persistent=pers, seed=12)
    checked = _check_engine(clo, oracle, r, layers=[0, 1])
    assert checked == {"persistent": 2, "offloaded": 2}
