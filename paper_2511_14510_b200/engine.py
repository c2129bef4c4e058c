"""Python mirror of the kvsim DecodeEngine API (engine.hpp:30-149) over the
C-ABI (include/clo.h). Same names and argument meaning as the reference:
EngineConfig / ModeFlags / DecodeEngine(cfg, profiles, plan, source) with
prefill(), decode_step(), run(), metrics(), head(l, g), collected_outputs(),
cache_state_json(), uniform_profiles(), layer0_only_plan().

B200 differences (documented in DESIGN.md): one engine serves `batch`
sequences (the reference runs one engine per sequence on a thread pool,
runner.cpp:186-278); decode_step is asynchronous (GPU-centric sync) and
state queries synchronise.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, ptr

Policy = {"similarity": _lib.POLICY_SIMILARITY, "lru": _lib.POLICY_LRU, "lfu": _lib.POLICY_LFU,
          "prefetch_only": _lib.POLICY_PREFETCH_ONLY}
Retriever = {"exact": _lib.RETRIEVER_EXACT, "sign_hash": _lib.RETRIEVER_SIGN_HASH}
KvDtype = {"bf16": _lib.DTYPE_BF16, "f32": _lib.DTYPE_F32}


@dataclass
class ModelShape:  # matrix.hpp:46-66
    num_layers: int = 0
    num_q_heads: int = 0
    num_kv_heads: int = 0
    head_dim: int = 128
    bytes_per_element: int = 2

    def group_size(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    def kv_group_of(self, q_head: int) -> int:
        return q_head // self.group_size()

    def first_q_head(self, kv_head: int) -> int:
        return kv_head * self.group_size()


@dataclass
class ModeFlags:  # engine.hpp:24-28
    always_miss: bool = False
    always_hit: bool = False
    tau_override: Optional[float] = None


@dataclass
class EngineConfig:  # engine.hpp:30-49 (+ B200 fields)
    shape: ModelShape = field(default_factory=ModelShape)
    k: int = 0
    sink_tokens: int = 4
    recent_tokens: int = 64
    retriever: str = "exact"
    hash_bits: int = 256
    retriever_seed: int = 1
    policy: str = "similarity"
    mode: ModeFlags = field(default_factory=ModeFlags)
    sync_override: Optional[int] = None
    collect_outputs: bool = False
    compute_oracle_error: bool = False
    # B200
    batch: int = 1
    kv_dtype: str = "bf16"
    kv_head_offset: int = 0
    device: int = 0
    victim_rows: int = -1  # HBM rows kept per offloaded head beyond the entry (-1: auto = 8k capped by free HBM, 0: none)

    def to_c(self, n_prompt: int, max_steps: int) -> _lib.EngineConfigC:
        c = _lib.EngineConfigC()
        _lib.load().clo_engine_config_defaults(C.byref(c))
        s = self.shape
        c.shape = _lib.ModelShape(s.num_layers, s.num_q_heads, s.num_kv_heads, s.head_dim,
                                  s.bytes_per_element)
        c.k, c.sink_tokens, c.recent_tokens = self.k, self.sink_tokens, self.recent_tokens
        if self.retriever not in Retriever:
            raise _lib.ConfigError(f"unknown retriever {self.retriever}")
        if self.policy not in Policy:
            raise _lib.ConfigError(f"unknown policy name: {self.policy}")
        c.retriever, c.hash_bits, c.retriever_seed = Retriever[self.retriever], self.hash_bits, self.retriever_seed
        c.policy = Policy[self.policy]
        c.always_miss, c.always_hit = int(self.mode.always_miss), int(self.mode.always_hit)
        c.has_tau_override = int(self.mode.tau_override is not None)
        c.tau_override = float(self.mode.tau_override or 0.0)
        c.sync_override = -1 if self.sync_override is None else int(self.sync_override)
        c.collect_outputs, c.compute_oracle_error = int(self.collect_outputs), int(self.compute_oracle_error)
        c.batch, c.n_prompt, c.max_steps = self.batch, n_prompt, max_steps
        c.kv_dtype, c.kv_head_offset, c.device = KvDtype[self.kv_dtype], self.kv_head_offset, self.device
        c.victim_rows = self.victim_rows
        return c


@dataclass
class HeadProfileEntry:  # head_profile.hpp:16-23
    q_importance: list
    kv_importance: float = 0.0
    s_hat: float = 0.0
    tau: float = -1.0
    difficulty: float = 0.0
    placement: str = "offloaded"


@dataclass
class PartitionPlan:  # head_profile.hpp:85-97 (persistent_heads per layer)
    layers: list  # list[list[int]]
    n_p: int = 0


def uniform_profiles(shape: ModelShape, tau: float):
    """engine.cpp:532-546."""
    return [[HeadProfileEntry(q_importance=[1.0] * shape.group_size(), kv_importance=1.0, s_hat=1.0,
                              tau=tau, difficulty=0.0) for _ in range(shape.num_kv_heads)]
            for _ in range(shape.num_layers)]


def layer0_only_plan(shape: ModelShape) -> PartitionPlan:
    """engine.cpp:548-555."""
    layers = [[] for _ in range(shape.num_layers)]
    layers[0] = list(range(shape.num_kv_heads))
    return PartitionPlan(layers=layers)


def profiles_from_arrays(tau: np.ndarray, q_importance: np.ndarray):
    L, H = tau.shape
    return [[HeadProfileEntry(q_importance=list(map(float, q_importance[l, g])), tau=float(tau[l, g]))
             for g in range(H)] for l in range(L)]


class HostKV:
    """Pinned, UVA-mapped host K/V store [B][Lk][H][nmax][d] (HeadStore::k/v).

    interleaved=True stores one buffer [B][Lk][H][nmax][2][d]: a token's K and
    V rows are contiguous (row stride 2d), so fetching it over PCIe touches one
    host page instead of two. `k` and `v` are strided views either way.
    numa_node >= 0 binds the pages to that host NUMA node (the one the gathering
    GPU's PCIe root hangs off, `device_numa_node`)."""

    def __init__(self, batch, layers, heads, nmax, d, kv_dtype, hugepages: bool = False,
                 interleaved: bool = False, numa_node: int = -1):
        lib = _lib.load()
        self.np_dtype = np.uint16 if kv_dtype == "bf16" else np.float32
        self.shape = (batch, layers, heads, nmax, d)
        self.interleaved = interleaved
        nbytes = int(np.prod(self.shape)) * np.dtype(self.np_dtype).itemsize
        self._ptrs = []
        arrays = []
        for _ in range(1 if interleaved else 2):
            p = C.c_void_p()
            size = 2 * nbytes if interleaved else nbytes
            # numa_node >= 0: pages bound to the GPU's host NUMA node (clo_host_alloc_numa)
            check(lib.clo_host_alloc_numa(size, _lib.HOST_HUGEPAGES if hugepages else 0, numa_node, C.byref(p)))
            self._ptrs.append(p.value)
            buf = (C.c_char * size).from_address(p.value)
            arrays.append(np.frombuffer(buf, dtype=self.np_dtype))
        if interleaved:
            kv = arrays[0].reshape(self.shape[:4] + (2, d))
            self.k, self.v = kv[..., 0, :], kv[..., 1, :]
        else:
            self.k, self.v = (a.reshape(self.shape) for a in arrays)
        el = np.dtype(self.np_dtype).itemsize
        self.strides = tuple(s // el for s in self.k.strides[:3])  # seq, layer, head (elements)
        self.row_stride = self.k.strides[3] // el

    def close(self):
        lib = _lib.load()
        for p in self._ptrs:
            lib.clo_host_free(p)
        self._ptrs = []

    def __del__(self):
        if getattr(self, "_ptrs", None):
            self.close()


def device_numa_node(device: int) -> int:
    """Host NUMA node of CUDA device `device`'s PCIe root (-1: not reported)."""
    lib = _lib.load()
    node = C.c_int(-1)
    check(lib.clo_device_numa_node(device, C.byref(node)))
    return node.value


def numa_node_cpus(node: int) -> set:
    """CPUs of host NUMA node `node` (sysfs cpulist), empty when unknown."""
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
    except OSError:
        return set()
    cpus = set()
    for part in filter(None, spec.split(",")):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus


class DecodeEngine:
    """DecodeEngine(cfg, profiles, plan, source) — engine.hpp:93-94.

    `source` is a SyntheticWorkload-like object (prompt_k/v, true_q, approx_q,
    new_k/v, step_new_kv). Host K/V lives in pinned memory owned here.
    """

    def __init__(self, cfg: EngineConfig, profiles, plan: PartitionPlan, source, host_kv=None):
        self.cfg, self.source = cfg, source
        s = cfg.shape
        L, H, m = s.num_layers, s.num_kv_heads, s.group_size()
        if len(profiles) != L:
            raise _lib.ArgumentError("profiles must cover every layer")
        for layer in profiles:
            if len(layer) != H:
                raise _lib.ArgumentError("profiles must cover every KV head")
            for e in layer:
                if len(e.q_importance) != m:
                    raise _lib.ArgumentError("profile importance width must equal the group size")
        if len(plan.layers) != L:
            raise _lib.ArgumentError("partition plan must cover every layer")
        tau = np.array([[e.tau for e in layer] for layer in profiles], np.float64)
        qimp = np.array([[e.q_importance for e in layer] for layer in profiles], np.float64)
        pers = np.zeros((L, H), np.int32)
        for l, heads in enumerate(plan.layers):
            for g in heads:
                if g < 0 or g >= H:
                    raise _lib.ArgumentError("partition plan names a KV head outside the model")
                pers[l, g] = 1
        self.n_prompt, self.steps = source.n_prompt, source.steps
        self.lib = _lib.load()
        c = cfg.to_c(self.n_prompt, self.steps)
        h = C.c_void_p()
        check(self.lib.clo_engine_create(C.byref(c), ptr(tau), ptr(qimp), ptr(pers), C.byref(h)))
        self.h = h.value
        nmax = self.n_prompt + self.steps
        Lk = 1 if getattr(source, "alias_layers", False) else L
        self.hkv = host_kv or HostKV(cfg.batch, Lk, H, nmax, s.head_dim, cfg.kv_dtype)
        if source.prompt_k is not None:  # None: the caller filled host_kv itself
            self.hkv.k[:, :, :, : self.n_prompt] = source.prompt_k
            self.hkv.v[:, :, :, : self.n_prompt] = source.prompt_v
        ss, ls, hs = self.hkv.strides
        check(self.lib.clo_engine_bind_host_kv_ex(self.h, self.hkv.k.ctypes.data, self.hkv.v.ctypes.data,
                                                  ss, 0 if Lk == 1 else ls, hs, self.hkv.row_stride))
        self.current_step = 0
        self._outputs = []
        self.world = 1

    def close(self):
        if getattr(self, "h", None):
            self.lib.clo_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # -- workflow -------------------------------------------------------------
    def prefill(self):
        q0 = np.ascontiguousarray(self.source.true_q[0], np.float32)
        check(self.lib.clo_prefill(self.h, ptr(q0), 1, None))

    def decode_step(self, timeline: bool = False):
        """One decode step; timeline=True also measures the per-layer
        LayerTiming breakdown (clo_engine_timeline_step)."""
        t = self.current_step + 1
        if t > self.source.steps:  # engine.cpp:226-228 (the C engine checks it too)
            raise _lib.ContractError("ContractError: decode_step past the end of the workload")
        tq = np.ascontiguousarray(self.source.true_q[t], np.float32)
        aq = np.ascontiguousarray(self.source.approx_q[t], np.float32)
        nk, nv = self.source.step_new_kv(t)
        s = self.cfg.shape
        out = np.empty((self.cfg.batch, s.num_layers, self.world * s.num_q_heads, s.head_dim), np.float32)
        io = _lib.StepIO(ptr(tq), ptr(aq), ptr(nk), ptr(nv), ptr(out), 1)
        step = self.lib.clo_engine_timeline_step if timeline else self.lib.clo_decode_step
        check(step(self.h, C.byref(io), None))
        check(self.lib.clo_engine_synchronize(self.h))
        self.current_step = t
        if self.cfg.collect_outputs:
            self._outputs.append(out)
        return out

    def run(self):
        self.prefill()
        for _ in range(self.source.steps):
            self.decode_step()

    # -- state ----------------------------------------------------------------
    def metrics(self) -> dict:
        mt = _lib.Metrics()
        check(self.lib.clo_get_metrics(self.h, C.byref(mt)))
        return {f: getattr(mt, f) for f, _ in _lib.Metrics._fields_}

    def sync_mode(self) -> int:
        return self.metrics()["sync_mode"]

    def head(self, layer: int, kv_head: int, seq: int = 0) -> dict:
        st = _lib.HeadState()
        idx = np.zeros(self.cfg.k, np.int32)
        hist = np.zeros(max(self.steps, 1), np.float64)
        check(self.lib.clo_get_head_state(self.h, seq, layer, kv_head, C.byref(st), ptr(idx), ptr(hist)))
        d = {f: getattr(st, f) for f, _ in _lib.HeadState._fields_}
        d["entry_indices"] = idx
        d["aggregated_history"] = hist[: st.n_history]
        return d

    def entry_rows(self, layer: int, kv_head: int, seq: int = 0):
        s = self.cfg.shape
        dt = np.uint16 if self.cfg.kv_dtype == "bf16" else np.float32
        k = np.zeros((self.cfg.k, s.head_dim), dt)
        v = np.zeros((self.cfg.k, s.head_dim), dt)
        check(self.lib.clo_get_entry_rows(self.h, seq, layer, kv_head, ptr(k), ptr(v)))
        return k, v

    def collected_outputs(self):
        """outputs[t][b][l] -> hq x d (engine.hpp:112-114, plus the batch axis)."""
        return self._outputs

    def cache_state_json(self, seq: int = 0) -> str:
        need = C.c_size_t()
        check(self.lib.clo_cache_state_json(self.h, seq, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(self.lib.clo_cache_state_json(self.h, seq, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def cache_state(self, seq: int = 0) -> dict:
        return json.loads(self.cache_state_json(seq))

    # -- KV-head sharding: fused head-output exchange (include/clo.h) ---------
    def exchange_handle(self, rank: int, world: int) -> bytes:
        """This engine's exchange handle (step 1 of the attach protocol)."""
        buf = (C.c_char * _lib.EXCHANGE_HANDLE_BYTES)()
        check(self.lib.clo_engine_exchange_handle(self.h, rank, world, buf))
        self._pending_world = world
        return bytes(buf)

    def attach_peers(self, handles) -> None:
        """Maps every rank's exchange buffer (handles in rank order); from the
        next step on, outputs cover the whole model's query heads."""
        blob = b"".join(handles)
        check(self.lib.clo_engine_attach_peers(self.h, blob))
        self.world = getattr(self, "_pending_world", len(handles))

    def timeline(self) -> dict:
        """DecodeEngine::timeline() (engine.hpp:105): PipelineTimeline of the
        steps run with timeline=True, measured on the device."""
        L = self.cfg.shape.num_layers
        per = (_lib.LayerTiming * L)()
        tot = _lib.LayerTiming()
        steps = C.c_uint64()
        check(self.lib.clo_get_timeline(self.h, per, L, C.byref(tot), C.byref(steps)))
        row = lambda t: {f: getattr(t, f) for f, _ in _lib.LayerTiming._fields_}
        return {"steps": steps.value, "per_layer": [row(t) for t in per], "totals": row(tot)}

    def timeline_spans(self) -> list:
        """(name, layer, start_ms, end_ms) of every kernel of the last timeline step."""
        cnt = C.c_int()
        check(self.lib.clo_timeline_spans(self.h, None, 0, C.byref(cnt)))
        buf = (_lib.KernelSpan * max(1, cnt.value))()
        check(self.lib.clo_timeline_spans(self.h, buf, cnt.value, C.byref(cnt)))
        return [(s.name.decode(), s.layer, s.start_ms, s.end_ms) for s in buf[:cnt.value]]

    def timeline_json(self) -> str:
        need = C.c_size_t()
        check(self.lib.clo_timeline_json(self.h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(self.lib.clo_timeline_json(self.h, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def kernel_launches(self) -> int:
        return self.lib.clo_engine_kernel_launches(self.h)

    def kernels_per_step(self) -> int:
        return self.lib.clo_engine_kernels_per_step(self.h)
