"""Head profiling and partition planning (profiler.cpp:19-125,
head_profile.cpp:17-154), over libclo (include/clo.h clo_profile_heads,
clo_plan_partition). The probe workloads are traces (trace.Trace); the
full / streaming / top-k attention of the importance fit runs on the GPU.

    profiles = profile_heads(["probe0.bin", "probe1.bin"], topk=64)
    plan = plan_partition(profiles, t_comp_s=5e-5, pcie_bw=5e10, mem_head_bytes=2*k*d*2)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check
from .engine import HeadProfileEntry, PartitionPlan
from .trace import Trace


def profile_heads(sources, blend_sequences: int = 1, blend_steps: int = 8, topk: int = 1,
                  sink_tokens: int = 4, recent_tokens: int = 64, eta: float = 0.8, p: float = 3.0,
                  epsilon: float = 0.1, provided_importance=None):
    """profile_heads (profiler.cpp:19-125) -> profiles[layer][kv_head] (HeadProfileEntry).
    provided_importance [L][hkv][m] replaces the blend fit (read_importance)."""
    lib = _lib.load()
    traces = [s if isinstance(s, Trace) else Trace(s) for s in sources]
    if not traces:
        raise _lib.ArgumentError("ArgumentError: profiling needs at least one probe workload")
    sh = traces[0].shape
    L, H, m = sh.num_layers, sh.num_kv_heads, sh.num_q_heads // sh.num_kv_heads
    cfg = _lib.ProfilerConfig()
    lib.clo_profiler_config_defaults(C.byref(cfg))
    cfg.blend_sequences, cfg.blend_steps, cfg.topk = blend_sequences, blend_steps, topk
    cfg.sink_tokens, cfg.recent_tokens = sink_tokens, recent_tokens
    cfg.eta, cfg.p, cfg.epsilon = eta, p, epsilon
    handles = (C.c_void_p * len(traces))(*[t.h for t in traces])
    out = (_lib.HeadProfileC * (L * H))()
    prov = None
    if provided_importance is not None:
        prov = np.ascontiguousarray(provided_importance, np.float64)
        if prov.shape != (L, H, m):
            raise _lib.ConfigError("ConfigError: provided importance must be [layer][kv_head][group]")
    check(lib.clo_profile_heads(handles, len(traces), C.byref(cfg), None if prov is None else prov.ctypes.data, out))
    return [[HeadProfileEntry(q_importance=list(out[l * H + g].q_importance[:m]),
                              kv_importance=out[l * H + g].kv_importance, s_hat=out[l * H + g].s_hat,
                              tau=out[l * H + g].tau, difficulty=out[l * H + g].difficulty)
             for g in range(H)] for l in range(L)]


def plan_partition(profiles, t_comp_s: float, pcie_bw: float, mem_head_bytes: float,
                   persist_bytes_per_head: int = 0, hbm_budget_bytes: int = 0):
    """plan_partition (head_profile.cpp:80-154): layer 0 all persistent, then the
    N_p = floor(t_comp * bw / mem_head) most difficult positive-difficulty heads
    per layer, within the HBM budget. Returns (PartitionPlan, n_p, n_dropped)."""
    lib = _lib.load()
    L, H = len(profiles), len(profiles[0])
    diff = np.array([[e.difficulty for e in layer] for layer in profiles], np.float64)
    pers = np.zeros((L, H), np.int32)
    n_p, nd = C.c_int(), C.c_int()
    check(lib.clo_plan_partition(diff.ctypes.data, L, H, t_comp_s, pcie_bw, float(mem_head_bytes),
                                 int(persist_bytes_per_head), int(hbm_budget_bytes), pers.ctypes.data,
                                 C.byref(n_p), C.byref(nd)))
    for l in range(L):
        for g in range(H):
            profiles[l][g].placement = "persistent" if pers[l, g] else "offloaded"
    return PartitionPlan(layers=[[g for g in range(H) if pers[l, g]] for l in range(L)]), n_p.value, nd.value
