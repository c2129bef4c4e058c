"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so (the C restatement, clo_oracle.c) and
`Reference` wraps oracle/_ref/libkvsim_ref.so (the unmodified reference kvsim
library compiled in place, via ref_shim.cpp). Both expose the same method
names so tests can run one check against either. Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs import this module; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkvsim_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_up = C.POINTER(C.c_uint64)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class EngineCfg(C.Structure):
    """Mirrors orc_engine_cfg / ref_engine_cfg (engine.hpp:30-49 subset)."""

    _fields_ = [
        ("num_layers", C.c_int), ("num_q_heads", C.c_int), ("num_kv_heads", C.c_int),
        ("head_dim", C.c_int), ("bytes_per_element", C.c_int),
        ("k", C.c_int), ("sink_tokens", C.c_int), ("recent_tokens", C.c_int),
        ("retriever", C.c_int), ("hash_bits", C.c_int), ("retriever_seed", C.c_uint64),
        ("policy", C.c_int), ("always_miss", C.c_int), ("always_hit", C.c_int),
        ("has_tau_override", C.c_int), ("tau_override", C.c_double),
        ("n_prompt", C.c_int), ("steps", C.c_int),
    ]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile liboracle.so (always) and _ref (when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class _Common:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, code):
        if code:
            raise OracleError(code, self._fn("last_error")().decode())

    # -- similarity cache ---------------------------------------------------
    def aggregate_similarity(self, sims, weights):
        sims = np.ascontiguousarray(sims, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        out = C.c_double()
        self._check(self._fn("aggregate_similarity")(_p(sims, C.c_double), _p(w, C.c_double),
                                                      C.c_int(len(sims)), C.byref(out)))
        return out.value

    def lookup(self, labels, label_valid, queries, weights, tau):
        """Returns (hit, aggregated, sims, reason, labels', valid')."""
        labels = np.array(labels, np.float64, order="C")
        valid = np.array(label_valid, np.int32)
        q = np.ascontiguousarray(queries, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        m, d = q.shape
        hit, reason = C.c_int(), C.c_int()
        agg = C.c_double()
        sims = np.zeros(m, np.float64)
        self._check(self._fn("lookup")(_p(labels, C.c_double), _p(valid, C.c_int),
                                        _p(q, C.c_double), _p(w, C.c_double), C.c_int(m),
                                        C.c_int(d), C.c_double(tau), C.byref(hit), C.byref(agg),
                                        _p(sims, C.c_double), C.byref(reason)))
        return bool(hit.value), agg.value, sims, reason.value, labels, valid

    # -- retrieval ------------------------------------------------------------
    def merge_group_topk(self, proposals, k):
        sizes = np.array([len(p) for p in proposals], np.int32)
        idx = np.array([i for p in proposals for i, _ in p], np.int32)
        sc = np.array([s for p in proposals for _, s in p], np.float64)
        out = np.zeros(k, np.int32)
        self._check(self._fn("merge_group_topk")(_p(sizes, C.c_int), C.c_int(len(sizes)),
                                                  _p(idx, C.c_int), _p(sc, C.c_double),
                                                  C.c_int(k), _p(out, C.c_int)))
        return out

    def topk_select_exact(self, q, keys, k):
        q = np.ascontiguousarray(q, np.float64)
        keys = np.ascontiguousarray(keys, np.float64)
        out = np.zeros(k, np.int32)
        self._check(self._fn("topk_select_exact")(_p(q, C.c_double), _p(keys, C.c_double),
                                                   C.c_int(keys.shape[0]), C.c_int(keys.shape[1]),
                                                   C.c_int(k), _p(out, C.c_int)))
        return out

    def topk_attention(self, q, keys, values, idx):
        q = np.ascontiguousarray(q, np.float64)
        keys = np.ascontiguousarray(keys, np.float64)
        values = np.ascontiguousarray(values, np.float64)
        idx = np.ascontiguousarray(idx, np.int32)
        out = np.zeros(keys.shape[1], np.float64)
        self._check(self._fn("topk_attention")(_p(q, C.c_double), _p(keys, C.c_double),
                                                _p(values, C.c_double), C.c_int(keys.shape[0]),
                                                C.c_int(keys.shape[1]), _p(idx, C.c_int),
                                                C.c_int(len(idx)), _p(out, C.c_double)))
        return out

    def sink_recent_indices(self, n, sink, recent):
        out = np.zeros(max(0, min(n, sink)) + max(0, min(n, recent)) + 1, np.int32)
        cnt, cl = C.c_int(), C.c_int()
        self._check(self._fn("sink_recent_indices")(C.c_int(n), C.c_int(sink), C.c_int(recent),
                                                     _p(out, C.c_int), C.byref(cnt), C.byref(cl)))
        return out[: cnt.value], bool(cl.value)

    def compute_threshold(self, s, eta=0.8, p=3.0):
        out = C.c_double()
        self._check(self._fn("compute_threshold")(C.c_double(s), C.c_double(eta), C.c_double(p),
                                                   C.byref(out)))
        return out.value

    def plan_partition(self, difficulty, t_comp_s, pcie_bw, mem_head_bytes,
                       persist_bytes_per_head=0, hbm_budget_bytes=0):
        diff = np.ascontiguousarray(difficulty, np.float64)
        L, H = diff.shape
        out = np.zeros((L, H), np.int32)
        n_p, nd = C.c_int(), C.c_int()
        self._check(self._fn("plan_partition")(_p(diff, C.c_double), C.c_int(L), C.c_int(H),
                                                C.c_double(t_comp_s), C.c_double(pcie_bw),
                                                C.c_double(mem_head_bytes),
                                                C.c_uint64(persist_bytes_per_head),
                                                C.c_uint64(hbm_budget_bytes), _p(out, C.c_int),
                                                C.byref(n_p), C.byref(nd)))
        return out.astype(bool), n_p.value, nd.value

    def cache_bytes(self, offloaded, entry_k, held, L, hq, d, e):
        f = self._fn("cache_bytes")
        f.restype = C.c_uint64
        return f(offloaded, entry_k, held, L, hq, d, e)

    def fill_normal(self, seed, n):
        out = np.zeros(n, np.float64)
        self._fn("fill_normal")(C.c_uint64(seed), _p(out, C.c_double), C.c_size_t(n))
        return out


class Oracle(_Common):
    """The C restatement (clo_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        super().__init__(path)
        self.lib.orc_engine_create.restype = C.c_void_p
        self.lib.orc_mix_seed3.restype = C.c_uint64

    def mix_seed3(self, base, a, b):
        return self.lib.orc_mix_seed3(C.c_uint64(base), C.c_uint64(a), C.c_uint64(b))

    def cosine_similarity(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        v = C.c_double()
        deg = self.lib.orc_cosine_similarity(_p(a, C.c_double), _p(b, C.c_double), C.c_int(len(a)),
                                             C.byref(v))
        return v.value, bool(deg)

    def encode_sign_hash(self, keys, hash_bits, seed):
        keys = np.ascontiguousarray(keys, np.float64)
        n, d = keys.shape
        proj = np.zeros((hash_bits, d), np.float64)
        bits = np.zeros((n, (hash_bits + 63) // 64), np.uint64)
        self._check(self.lib.orc_encode_sign_hash(_p(keys, C.c_double), C.c_int(n), C.c_int(d),
                                                  C.c_int(hash_bits), C.c_uint64(seed),
                                                  _p(proj, C.c_double), _p(bits, C.c_uint64)))
        return proj, bits

    def retrieve_scored(self, q, keys, k, variant=0, hash_bits=256, seed=0):
        q = np.ascontiguousarray(q, np.float64)
        keys = np.ascontiguousarray(keys, np.float64)
        n, d = keys.shape
        idx = np.zeros(k, np.int32)
        sc = np.zeros(k, np.float64)
        if variant == 0:
            proj = np.zeros(1)
            bits = np.zeros(1, np.uint64)
        else:
            proj, bits = self.encode_sign_hash(keys, hash_bits, seed)
        self._check(self.lib.orc_retrieve_scored(_p(q, C.c_double), C.c_int(d), C.c_int(variant),
                                                 _p(keys, C.c_double), _p(proj, C.c_double),
                                                 _p(bits, C.c_uint64), C.c_int(hash_bits),
                                                 C.c_int(n), C.c_int(k), _p(idx, C.c_int),
                                                 _p(sc, C.c_double)))
        return idx, sc

    # -- engine ---------------------------------------------------------------
    def engine(self, cfg: EngineCfg, tau, q_importance, persistent, prompt_k, prompt_v):
        return OracleEngine(self, cfg, tau, q_importance, persistent, prompt_k, prompt_v)


class OrcHeadState(C.Structure):
    _fields_ = [
        ("hits", C.c_uint64), ("misses", C.c_uint64), ("transferred_bytes", C.c_uint64),
        ("persistent_bytes", C.c_uint64), ("last_update_step", C.c_int),
        ("entry_last_update_step", C.c_int), ("labels_valid", C.c_int),
        ("window_held_tokens", C.c_int), ("persistent", C.c_int), ("n_history", C.c_int),
    ]


class OracleEngine:
    """DecodeEngine restatement for one sequence (engine.cpp:106-415)."""

    def __init__(self, orc: Oracle, cfg, tau, q_importance, persistent, prompt_k, prompt_v):
        self.o, self.cfg = orc, cfg
        tau = np.ascontiguousarray(tau, np.float64)
        qi = np.ascontiguousarray(q_importance, np.float64)
        pers = np.ascontiguousarray(persistent, np.int32)
        pk = np.ascontiguousarray(prompt_k, np.float64)
        pv = np.ascontiguousarray(prompt_v, np.float64)
        st = C.c_int()
        self.h = orc.lib.orc_engine_create(C.byref(cfg), _p(tau, C.c_double), _p(qi, C.c_double),
                                           _p(pers, C.c_int), _p(pk, C.c_double),
                                           _p(pv, C.c_double), C.byref(st))
        if not self.h:
            orc._check(st.value)

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_engine_destroy(C.c_void_p(self.h))
            self.h = None

    def prefill(self, true_q0):
        q = np.ascontiguousarray(true_q0, np.float64)
        self.o._check(self.o.lib.orc_engine_prefill(C.c_void_p(self.h), _p(q, C.c_double)))

    def decode_step(self, true_q, approx_q, new_k, new_v):
        c = self.cfg
        out = np.zeros((c.num_layers, c.num_q_heads, c.head_dim), np.float64)
        tq = np.ascontiguousarray(true_q, np.float64)
        aq = np.ascontiguousarray(approx_q, np.float64)
        nk = np.ascontiguousarray(new_k, np.float64)
        nv = np.ascontiguousarray(new_v, np.float64)
        self.o._check(self.o.lib.orc_engine_decode_step(C.c_void_p(self.h), _p(tq, C.c_double),
                                                        _p(aq, C.c_double), _p(nk, C.c_double),
                                                        _p(nv, C.c_double), _p(out, C.c_double)))
        return out

    def head_state(self, l, g):
        c = self.cfg
        st = OrcHeadState()
        idx = np.zeros(c.k, np.int32)
        hist = np.zeros(max(c.steps, 1), np.float64)
        ek = np.zeros((c.k, c.head_dim), np.float64)
        ev = np.zeros((c.k, c.head_dim), np.float64)
        self.o._check(self.o.lib.orc_engine_head_state(C.c_void_p(self.h), l, g, C.byref(st),
                                                       _p(idx, C.c_int), _p(hist, C.c_double),
                                                       _p(ek, C.c_double), _p(ev, C.c_double)))
        return {
            "hits": st.hits, "misses": st.misses, "transferred_bytes": st.transferred_bytes,
            "persistent_served_bytes": st.persistent_bytes,
            "last_update_step": st.last_update_step,
            "entry_last_update_step": st.entry_last_update_step,
            "labels_valid": st.labels_valid, "window_held_tokens": st.window_held_tokens,
            "persistent": bool(st.persistent), "entry_indices": idx,
            "aggregated_history": hist[: st.n_history], "entry_k": ek, "entry_v": ev,
        }


class Reference(_Common):
    """The unmodified reference library (oracle/_ref/libkvsim_ref.so)."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        super().__init__(path)
        self.lib.ref_mix_seed3.restype = C.c_uint64

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def mix_seed3(self, base, a, b):
        return self.lib.ref_mix_seed3(C.c_uint64(base), C.c_uint64(a), C.c_uint64(b))

    def cosine_similarity(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        v, deg = C.c_double(), C.c_int()
        self._check(self.lib.ref_cosine_similarity(_p(a, C.c_double), _p(b, C.c_double),
                                                   C.c_int(len(a)), C.byref(v), C.byref(deg)))
        return v.value, bool(deg.value)

    def encode_sign_hash(self, keys, hash_bits, seed):
        keys = np.ascontiguousarray(keys, np.float64)
        n, d = keys.shape
        proj = np.zeros((hash_bits, d), np.float64)
        bits = np.zeros((n, (hash_bits + 63) // 64), np.uint64)
        self._check(self.lib.ref_encode_sign_hash(_p(keys, C.c_double), C.c_int(n), C.c_int(d),
                                                  C.c_int(hash_bits), C.c_uint64(seed),
                                                  _p(proj, C.c_double), _p(bits, C.c_uint64)))
        return proj, bits

    def retrieve_scored(self, q, keys, k, variant=0, hash_bits=256, seed=0):
        q = np.ascontiguousarray(q, np.float64)
        keys = np.ascontiguousarray(keys, np.float64)
        n, d = keys.shape
        idx = np.zeros(k, np.int32)
        sc = np.zeros(k, np.float64)
        self._check(self.lib.ref_retrieve_scored(_p(q, C.c_double), C.c_int(d), C.c_int(variant),
                                                 _p(keys, C.c_double), C.c_int(n), C.c_int(k),
                                                 C.c_int(hash_bits), C.c_uint64(seed),
                                                 _p(idx, C.c_int), _p(sc, C.c_double)))
        return idx, sc

    # -- trace wire format (trace_io.cpp) -----------------------------------
    def record_synthetic_trace(self, path, L, hq, hkv, d, n_prompt, steps, d_model=64, sigma_step=0.02,
                               sigma_layer=0.01, seed=1, tie=False, width=8):
        """The reference's SyntheticModel recorded with record_trace + write_trace."""
        self._check(self.lib.ref_record_synthetic_trace(
            C.c_int(L), C.c_int(hq), C.c_int(hkv), C.c_int(d), C.c_int(d_model), C.c_int(n_prompt),
            C.c_int(steps), C.c_double(sigma_step), C.c_double(sigma_layer), C.c_uint64(seed),
            C.c_int(int(tie)), C.c_int(width), str(path).encode()))

    def read_trace(self, path):
        """read_trace(path) -> (hdr, prompt [L][H][2][n][d], hidden [S+1][L][hq*d], step [S][L][2][H][d])."""
        hdr = np.zeros(7, np.int32)
        self._check(self.lib.ref_read_trace(str(path).encode(), _p(hdr, C.c_int), None, None, None))
        L, hq, H, d, n, S, _ = (int(x) for x in hdr)
        prompt = np.zeros((L, H, 2, n, d))
        hidden = np.zeros((S + 1, L, hq * d))
        step = np.zeros((max(S, 0), L, 2, H, d))
        self._check(self.lib.ref_read_trace(str(path).encode(), _p(hdr, C.c_int), _p(prompt, C.c_double),
                                            _p(hidden, C.c_double), _p(step, C.c_double)))
        return hdr, prompt, hidden, step

    def profile_heads(self, paths, blend_sequences=1, blend_steps=8, topk=1, sink=4, recent=64, eta=0.8, p=3.0,
                      epsilon=0.1, provided=None):
        """profile_heads over TraceSources: dict of q_importance [L][H][m], kv_importance, s_hat, tau,
        difficulty [L][H]."""
        hdr = self.read_trace(paths[0])[0]
        L, hq, H = int(hdr[0]), int(hdr[1]), int(hdr[2])
        m = hq // H
        arr = (C.c_char_p * len(paths))(*[str(x).encode() for x in paths])
        qi = np.zeros((L, H, m))
        out = {k: np.zeros((L, H)) for k in ("kv_importance", "s_hat", "tau", "difficulty")}
        prov = None if provided is None else np.ascontiguousarray(provided, np.float64)
        self._check(self.lib.ref_profile_heads(
            arr, C.c_int(len(paths)), C.c_int(blend_sequences), C.c_int(blend_steps), C.c_int(topk), C.c_int(sink),
            C.c_int(recent), C.c_double(eta), C.c_double(p), C.c_double(epsilon),
            None if prov is None else _p(prov, C.c_double), _p(qi, C.c_double),
            *[_p(out[k], C.c_double) for k in ("kv_importance", "s_hat", "tau", "difficulty")]))
        out["q_importance"] = qi
        return out

    def run_engine_trace(self, cfg: EngineCfg, tau, q_importance, persistent, path, json_cap=1 << 24):
        """Reference DecodeEngine over TraceSource(read_trace(path)): (outputs, cache_state_json)."""
        tau_ = np.ascontiguousarray(tau, np.float64)
        qi = np.ascontiguousarray(q_importance, np.float64)
        pers = np.ascontiguousarray(persistent, np.int32)
        outs = np.zeros((max(cfg.steps, 1), cfg.num_layers, cfg.num_q_heads, cfg.head_dim))
        buf = C.create_string_buffer(json_cap)
        self._check(self.lib.ref_run_engine_trace(
            C.byref(cfg), _p(tau_, C.c_double), _p(qi, C.c_double), _p(pers, C.c_int), str(path).encode(),
            _p(outs, C.c_double), buf, C.c_size_t(json_cap)))
        return outs, buf.value.decode()

    def set_compute_oracle_error(self, on: bool) -> None:
        """EngineConfig::compute_oracle_error (engine.hpp:48) for the following engine runs."""
        self.lib.ref_set_compute_oracle_error(int(on))

    def run_engine(self, cfg: EngineCfg, tau, q_importance, persistent, prompt_k, prompt_v,
                   true_q, approx_q, new_k, new_v, json_cap=1 << 24):
        """Full reference DecodeEngine run; returns (outputs, cache_state_json, step_seconds)."""
        arrs = [np.ascontiguousarray(a, np.float64) for a in
                (tau, q_importance, prompt_k, prompt_v, true_q, approx_q, new_k, new_v)]
        pers = np.ascontiguousarray(persistent, np.int32)
        outs = np.zeros((max(cfg.steps, 1), cfg.num_layers, cfg.num_q_heads, cfg.head_dim))
        buf = C.create_string_buffer(json_cap)
        secs = np.zeros(max(cfg.steps, 1), np.float64)
        tau_, qi, pk, pv, tq, aq, nk, nv = arrs
        self._check(self.lib.ref_run_engine(
            C.byref(cfg), _p(tau_, C.c_double), _p(qi, C.c_double), _p(pers, C.c_int),
            _p(pk, C.c_double), _p(pv, C.c_double), _p(tq, C.c_double), _p(aq, C.c_double),
            _p(nk, C.c_double), _p(nv, C.c_double), _p(outs, C.c_double), buf,
            C.c_size_t(json_cap), _p(secs, C.c_double)))
        return outs[: cfg.steps], buf.value.decode(), secs[: cfg.steps]

    def bench_units(self, cfg: EngineCfg, tau, q_importance, prompt_k, prompt_v, true_q,
                    approx_q, new_k, new_v, threads, warmup=0):
        """`threads` independent engines, each one (layer, kv head) unit; tau
        [threads] and q_importance [threads][m]: thread w's head profile
        (scalars / one row are broadcast to every thread)."""
        tau_ = np.ascontiguousarray(np.broadcast_to(np.asarray(tau, np.float64), (threads,)))
        m = cfg.num_q_heads
        qi = np.ascontiguousarray(np.broadcast_to(np.asarray(q_importance, np.float64).reshape(-1, m), (threads, m)))
        arrs = [np.ascontiguousarray(a, np.float64) for a in
                (prompt_k, prompt_v, true_q, approx_q, new_k, new_v)]
        pk, pv, tq, aq, nk, nv = arrs
        sps = np.zeros(threads)
        pre = np.zeros(threads)
        self._check(self.lib.ref_bench_units(
            C.byref(cfg), _p(tau_, C.c_double), _p(qi, C.c_double), _p(pk, C.c_double),
            _p(pv, C.c_double), _p(tq, C.c_double), _p(aq, C.c_double), _p(nk, C.c_double),
            _p(nv, C.c_double), C.c_int(threads), C.c_int(warmup), _p(sps, C.c_double),
            _p(pre, C.c_double)))
        return sps, pre
