"""Shared harness: run the CUDA engine and the CPU oracle engine on the same
synthetic workload and compare everything the reference exposes
(the GPU analogue of acceptance criterion 4, acceptance_main.cpp:142-206)."""
from __future__ import annotations

import numpy as np

from oracle.bind import EngineCfg
from paper_2511_14510_b200 import (DecodeEngine, EngineConfig, HostKV, ModeFlags, ModelShape,
                                   PartitionPlan, profiles_from_arrays)
from paper_2511_14510_b200.workload import Shape, SyntheticWorkload, widen

POLICY_CODE = {"similarity": 0, "prefetch_only": 3}


def make_case(L=3, hq=4, hkv=2, d=16, n_prompt=96, steps=12, k=8, batch=2, kv_dtype="f32",
              retriever="sign_hash", policy="similarity", sink=2, recent=8, always_miss=False,
              always_hit=False, tau_override=None, persistent=None, seed=5, sigma_step=0.15,
              hash_bits=256, alias_layers=False, tau=None, interleaved=False, victim_rows=-1):
    shape = Shape(L, hq, hkv, d)
    wl = SyntheticWorkload(shape, batch, n_prompt, steps, kv_dtype=kv_dtype, sigma_step=sigma_step,
                           seed=seed, alias_layers=alias_layers)
    rng = np.random.default_rng(seed + 100)
    m = hq // hkv
    qimp = rng.uniform(0.0, 1.0, (L, hkv, m))
    if tau is None:
        tau = rng.uniform(0.5, 0.95, (L, hkv))
    tau = np.broadcast_to(np.asarray(tau, np.float64), (L, hkv)).copy()
    if persistent is None:
        persistent = np.zeros((L, hkv), np.int32)
        persistent[0] = 1
    cfg = EngineConfig(shape=ModelShape(L, hq, hkv, d, 2 if kv_dtype == "bf16" else 4), k=k,
                       sink_tokens=sink, recent_tokens=recent, retriever=retriever,
                       hash_bits=hash_bits, retriever_seed=11, policy=policy,
                       mode=ModeFlags(always_miss, always_hit, tau_override), collect_outputs=True,
                       batch=batch, kv_dtype=kv_dtype, victim_rows=victim_rows)
    plan = PartitionPlan(layers=[[g for g in range(hkv) if persistent[l, g]] for l in range(L)])
    return dict(shape=shape, wl=wl, cfg=cfg, plan=plan, tau=tau, qimp=qimp,
                persistent=np.asarray(persistent, np.int32), interleaved=interleaved)


def oracle_cfg(case) -> EngineCfg:
    cfg, wl = case["cfg"], case["wl"]
    s = cfg.shape
    c = EngineCfg()
    c.num_layers, c.num_q_heads, c.num_kv_heads = s.num_layers, s.num_q_heads, s.num_kv_heads
    c.head_dim, c.bytes_per_element = s.head_dim, s.bytes_per_element
    c.k, c.sink_tokens, c.recent_tokens = cfg.k, cfg.sink_tokens, cfg.recent_tokens
    c.retriever = 0 if cfg.retriever == "exact" else 1
    c.hash_bits, c.retriever_seed = cfg.hash_bits, cfg.retriever_seed
    c.policy = POLICY_CODE[cfg.policy]
    c.always_miss, c.always_hit = int(cfg.mode.always_miss), int(cfg.mode.always_hit)
    c.has_tau_override = int(cfg.mode.tau_override is not None)
    c.tau_override = float(cfg.mode.tau_override or 0.0)
    c.n_prompt, c.steps = wl.n_prompt, wl.steps
    return c


def gpu_engine(case) -> DecodeEngine:
    hkv = None
    if case.get("interleaved"):  # host K|V rows of a token contiguous (row stride 2d)
        cfg, wl = case["cfg"], case["wl"]
        s = cfg.shape
        Lk = 1 if getattr(wl, "alias_layers", False) else s.num_layers
        hkv = HostKV(cfg.batch, Lk, s.num_kv_heads, wl.n_prompt + wl.steps, s.head_dim, cfg.kv_dtype,
                     interleaved=True)
    return DecodeEngine(case["cfg"], profiles_from_arrays(case["tau"], case["qimp"]), case["plan"],
                        case["wl"], host_kv=hkv)


def oracle_engines(case, oracle):
    wl = case["wl"]
    engines = []
    for b in range(wl.batch):
        pk, pv, tq, aq, nk, nv = wl.oracle_inputs(b)
        e = oracle.engine(oracle_cfg(case), case["tau"], case["qimp"], case["persistent"], pk, pv)
        engines.append((e, tq, aq, nk, nv))
    return engines


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    den = np.sqrt((want * want).sum(axis=-1))
    num = np.sqrt(((got - want) ** 2).sum(axis=-1))
    return np.where(den > 0, num / np.where(den > 0, den, 1), num)


class PoolModel:
    """The engine's HBM rows of one offloaded head (gather.cu reconcile): an
    entry area of k slots (the entry, in slot order) and a victim area of
    `victim` slots (8k when negative) holding rows that left the entry.
    New tokens in the entry area keep their slot; the others take the slots
    the leaving tokens free (ascending pairs), arriving from the victim area
    when resident there (promotion) else over PCIe; each leaving row is
    demoted into the victim area, a FIFO ring walked by a cursor (promotion
    sources skipped).
    reconcile() returns the rows fetched over PCIe."""

    def __init__(self, k, victim):
        self.k = k
        self.P = k + (8 * k if victim < 0 else victim)
        self.slot_tok = [-1] * self.P
        self.age = [-1] * self.P
        self.t2s = {}
        self.vh = 0  # FIFO cursor over the victim area

    def reconcile(self, new_sel, t, fresh=False):
        k = self.k
        new_sel = [int(x) for x in new_sel]
        kept, need = set(), []
        for i, tok in enumerate(new_sel):
            sl = self.t2s.get(tok)
            if sl is not None and sl < k:
                kept.add(sl)
            else:
                need.append(i)
        freed = [e for e in range(k) if e not in kept]
        prom = {self.t2s[new_sel[i]] for i in need if new_sel[i] in self.t2s}
        V = self.P - k
        ndem, dv = 0, []
        if not fresh and need and V > 0:  # FIFO ring from the cursor, skipping promotion sources
            W = min(V, len(need) + len(prom))
            cands = [(q, k + (self.vh + q) % V) for q in range(W) if k + (self.vh + q) % V not in prom]
            ndem = min(len(need), len(cands))
            dv = [p for _, p in cands[:ndem]]
            if ndem:
                self.vh = (self.vh + cands[ndem - 1][0] + 1) % V
        host = 0
        for j, pos in enumerate(need):
            e, tok = freed[j], new_sel[pos]
            x = self.slot_tok[e]
            sl = self.t2s.get(tok)
            if j < ndem and x >= 0:
                w = dv[j]
                y = self.slot_tok[w]
                if y >= 0:
                    del self.t2s[y]
                self.t2s[x] = w
                self.slot_tok[w] = x
                self.age[w] = t
            elif x >= 0:
                del self.t2s[x]
            if sl is not None:  # promotion: the victim slot empties
                self.slot_tok[sl] = -1
                self.age[sl] = -1
            else:
                host += 1
            self.t2s[tok] = e
            self.slot_tok[e] = tok
        return host


def run_and_compare(case, oracle, check_rows=True, tol=None):
    """Steps both engines in lockstep; asserts bit-exact selections, decisions,
    histories and gathered rows, and outputs within `tol` relative L2."""
    cfg, wl = case["cfg"], case["wl"]
    s = cfg.shape
    L, H = s.num_layers, s.num_kv_heads
    if tol is None:
        tol = 2e-2 if cfg.kv_dtype == "bf16" else 1e-3
    g_eng = gpu_engine(case)
    o_engs = oracle_engines(case, oracle)
    g_eng.prefill()
    for e, tq, *_ in o_engs:
        e.prefill(tq[0])
    worst = 0.0
    fetched_rows = 0  # rows the pooled delta gather moves over PCIe (not resident in the head's HBM pool)
    prev, pools = {}, {}
    for b in range(len(o_engs)):
        for l in range(L):
            for g in range(H):
                st0 = o_engs[b][0].head_state(l, g)
                if not st0["persistent"]:
                    prev[(b, l, g)] = (st0["misses"], set(map(int, st0["entry_indices"])))
                    pools[(b, l, g)] = PoolModel(cfg.k, cfg.victim_rows)
                    pools[(b, l, g)].reconcile(list(map(int, st0["entry_indices"])), 0, fresh=True)
    for t in range(1, wl.steps + 1):
        out = g_eng.decode_step()
        for b, (e, tq, aq, nk, nv) in enumerate(o_engs):
            want = e.decode_step(tq[t], aq[t], nk[t - 1], nv[t - 1])
            err = rel_l2(out[b], want)
            worst = max(worst, float(err.max()))
            for l in range(L):
                for g in range(H):
                    gs = g_eng.head(l, g, seq=b)
                    os_ = e.head_state(l, g)
                    where = f"step {t} seq {b} layer {l} head {g}"
                    assert gs["hits"] == os_["hits"], where
                    assert gs["misses"] == os_["misses"], where
                    assert gs["last_update_step"] == os_["last_update_step"], where
                    if not os_["persistent"]:
                        pm, pset = prev[(b, l, g)]
                        cur = set(map(int, os_["entry_indices"]))
                        if os_["misses"] > pm and cfg.policy == "similarity":
                            fetched_rows += pools[(b, l, g)].reconcile(list(map(int, os_["entry_indices"])), t)
                        prev[(b, l, g)] = (os_["misses"], cur)
                        assert gs["window_held_tokens"] == os_["window_held_tokens"], where
                        if cfg.policy == "similarity":
                            np.testing.assert_array_equal(gs["entry_indices"], os_["entry_indices"],
                                                          err_msg=where)
                            assert gs["entry_last_update_step"] == os_["entry_last_update_step"], where
                            assert gs["labels_valid"] == os_["labels_valid"], where
                            np.testing.assert_array_equal(gs["aggregated_history"],
                                                          os_["aggregated_history"], err_msg=where)
                            if check_rows:
                                kr, vr = g_eng.entry_rows(l, g, seq=b)
                                np.testing.assert_array_equal(widen(kr, cfg.kv_dtype), os_["entry_k"],
                                                              err_msg=where)
                                np.testing.assert_array_equal(widen(vr, cfg.kv_dtype), os_["entry_v"],
                                                              err_msg=where)
    assert worst <= tol, f"worst relative L2 {worst:.3g} > {tol}"
    if cfg.policy == "similarity":
        esz = 2 if cfg.kv_dtype == "bf16" else 4
        got = g_eng.metrics()["gathered_bytes_device"]
        assert got == fetched_rows * 2 * s.head_dim * esz, (got, fetched_rows)
    return g_eng, o_engs, worst
