"""Synthetic CLO decode workloads (inputs only; not part of the hot path).

A StepSource-shaped bundle (synthetic_model.hpp:16-28): prompt K/V per
(sequence, layer, KV head), per-step true and approximate queries, and per-step
new K/V rows. Queries follow the reference's drift-walk idea
(synthetic_model.cpp:22-27,108-176): q_t = normalize(q_{t-1} + sigma_step * g)
per (sequence, layer, query head); the approximate query of layer l is the true
query perturbed by a sigma_layer drift (a stand-in for "layer l-1 hidden state
through layer l's W_Q"). K/V rows are N(0,1) rounded to the storage dtype.

Everything is generated at storage precision (bf16 as uint16 bit patterns, or
float32) and widened EXACTLY to float64 for the CPU oracle, so the CUDA path
and the oracle consume identical values.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def widen(a: np.ndarray, kv_dtype: str) -> np.ndarray:
    """Storage values -> exact float64."""
    if kv_dtype == "bf16":
        return bf16_bits_to_f32(a).astype(np.float64)
    return np.asarray(a, np.float32).astype(np.float64)


def to_storage(x: np.ndarray, kv_dtype: str) -> np.ndarray:
    return f32_to_bf16_bits(x) if kv_dtype == "bf16" else np.ascontiguousarray(x, np.float32)


def _normalize(x: np.ndarray) -> np.ndarray:
    return x / np.linalg.norm(x, axis=-1, keepdims=True)


@dataclass
class Shape:
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int

    @property
    def group_size(self) -> int:
        return self.num_q_heads // self.num_kv_heads


class SyntheticWorkload:
    """Arrays (numpy) for `batch` sequences:
      prompt_k/v [B][Lk][H][n_prompt][d]   storage dtype (Lk = 1 when aliased)
      new_k/v    [steps][B][Lk][H][d]      storage dtype
      true_q     [steps+1][B][L][hq][d]    float32 (index 0 = prefill's step 0)
      approx_q   [steps+1][B][L][hq][d]    float32
    """

    def __init__(self, shape: Shape, batch: int, n_prompt: int, steps: int, kv_dtype: str = "bf16",
                 sigma_step: float = 0.05, sigma_layer: float = 0.01, seed: int = 1,
                 alias_layers: bool = False):
        self.shape, self.batch, self.n_prompt, self.steps = shape, batch, n_prompt, steps
        self.kv_dtype, self.alias_layers = kv_dtype, alias_layers
        rng = np.random.default_rng(seed)
        L, HQ, H, d = shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
        Lk = 1 if alias_layers else L
        self.prompt_k = to_storage(rng.standard_normal((batch, Lk, H, n_prompt, d), np.float32), kv_dtype)
        self.prompt_v = to_storage(rng.standard_normal((batch, Lk, H, n_prompt, d), np.float32), kv_dtype)
        self.new_k = to_storage(rng.standard_normal((steps, batch, Lk, H, d), np.float32), kv_dtype)
        self.new_v = to_storage(rng.standard_normal((steps, batch, Lk, H, d), np.float32), kv_dtype)
        q = _normalize(rng.standard_normal((batch, L, HQ, d)))
        tq = np.empty((steps + 1, batch, L, HQ, d), np.float32)
        aq = np.empty_like(tq)
        for t in range(steps + 1):
            if t:
                q = _normalize(q + sigma_step * rng.standard_normal(q.shape))
            tq[t] = q
            aq[t] = _normalize(q + sigma_layer * rng.standard_normal(q.shape))
        self.true_q, self.approx_q = tq, aq

    # -- per-step views in the engine's [B][L][...] layout -------------------
    def step_new_kv(self, t: int):
        """New K/V rows of decode step t (1-based) as [B][L][H][d] storage arrays."""
        k, v = self.new_k[t - 1], self.new_v[t - 1]
        if self.alias_layers:
            L = self.shape.num_layers
            k = np.ascontiguousarray(np.broadcast_to(k, (k.shape[0], L) + k.shape[2:]))
            v = np.ascontiguousarray(np.broadcast_to(v, (v.shape[0], L) + v.shape[2:]))
        return k, v

    # -- oracle (float64) views of one sequence -------------------------------
    def oracle_inputs(self, b: int):
        """(prompt_k, prompt_v [L][H][n][d], true_q, approx_q [(steps+1)][L][hq][d],
        new_k, new_v [steps][L][H][d]) widened to float64 for sequence b."""
        L = self.shape.num_layers
        pk = widen(self.prompt_k[b], self.kv_dtype)
        pv = widen(self.prompt_v[b], self.kv_dtype)
        nk = widen(self.new_k[:, b], self.kv_dtype)
        nv = widen(self.new_v[:, b], self.kv_dtype)
        if self.alias_layers:
            pk = np.repeat(pk, L, axis=0)
            pv = np.repeat(pv, L, axis=0)
            nk = np.repeat(nk, L, axis=1)
            nv = np.repeat(nv, L, axis=1)
        tq = self.true_q[:, b].astype(np.float64)
        aq = self.approx_q[:, b].astype(np.float64)
        return pk, pv, tq, aq, nk, nv


def synthetic_profiles(shape: Shape, seed: int = 7, eta: float = 0.8, p: float = 3.0,
                       threshold=None):
    """Per-head q_importance ~ U(0,1) and tau = compute_threshold(max over the
    group, eta, p) (head_profile.cpp:17-25; kv importance = group max,
    head_profile.hpp:70-75). `threshold(s, eta, p)` computes tau."""
    rng = np.random.default_rng(seed)
    L, H, m = shape.num_layers, shape.num_kv_heads, shape.group_size
    qimp = rng.uniform(0.0, 1.0, (L, H, m))
    tau = np.empty((L, H))
    for l in range(L):
        for g in range(H):
            tau[l, g] = threshold(float(qimp[l, g].max()), eta, p)
    return tau, qimp


class HeadSlice:
    """View of a SyntheticWorkload restricted to KV heads [kv0, kv0+n_kv) and
    their query heads (a KV-head shard, paper_2511_14510_b200/dist.py)."""

    def __init__(self, wl: SyntheticWorkload, kv0: int, n_kv: int, q0: int, n_q: int):
        self.shape = Shape(wl.shape.num_layers, n_q, n_kv, wl.shape.head_dim)
        self.batch, self.n_prompt, self.steps = wl.batch, wl.n_prompt, wl.steps
        self.kv_dtype, self.alias_layers = wl.kv_dtype, wl.alias_layers
        self.prompt_k = np.ascontiguousarray(wl.prompt_k[:, :, kv0:kv0 + n_kv])
        self.prompt_v = np.ascontiguousarray(wl.prompt_v[:, :, kv0:kv0 + n_kv])
        self.new_k = np.ascontiguousarray(wl.new_k[:, :, :, kv0:kv0 + n_kv])
        self.new_v = np.ascontiguousarray(wl.new_v[:, :, :, kv0:kv0 + n_kv])
        self.true_q = np.ascontiguousarray(wl.true_q[:, :, :, q0:q0 + n_q])
        self.approx_q = np.ascontiguousarray(wl.approx_q[:, :, :, q0:q0 + n_q])

    step_new_kv = SyntheticWorkload.step_new_kv
