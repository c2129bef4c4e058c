"""Workload traces in the reference's wire format (trace_io.hpp:12-64,
trace_io.cpp:83-266), read and written by libclo (include/clo.h clo_trace_*).

TraceSource mirrors kvsim::TraceSource (prompt_tokens, decode_steps,
prompt_k/v, true_query, approx_query, new_k_row, new_v_row) and also exposes
the batched arrays DecodeEngine consumes, so a trace recorded by the
reference replays on the GPU engine:

    src = TraceSource(["seq0.bin", "seq1.bin"], kv_dtype="f32")
    eng = DecodeEngine(cfg, profiles, plan, src); eng.run()

A trace holds one sequence; a list of traces with one shape is a batch.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check
from .workload import Shape

_DT = {"bf16": (_lib.DTYPE_BF16, np.uint16), "f32": (_lib.DTYPE_F32, np.float32), "f64": (_lib.DTYPE_F64, np.float64)}


class Trace:
    """One opened trace file (read_trace)."""

    def __init__(self, path: str):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.clo_trace_open(str(path).encode(), C.byref(h)))
        self.h = h.value
        s = _lib.ModelShape()
        n, st, w = C.c_int(), C.c_int(), C.c_int()
        check(self.lib.clo_trace_info(self.h, C.byref(s), C.byref(n), C.byref(st), C.byref(w)))
        self.shape = Shape(s.num_layers, s.num_q_heads, s.num_kv_heads, s.head_dim)
        self.n_prompt, self.n_steps, self.element_width = n.value, st.value, w.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.clo_trace_close(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def prompt(self, layer: int, kv_head: int, kv_dtype: str = "f64"):
        code, npdt = _DT[kv_dtype]
        k = np.empty((self.n_prompt, self.shape.head_dim), npdt)
        v = np.empty_like(k)
        check(self.lib.clo_trace_prompt(self.h, layer, kv_head, code, k.ctypes.data, v.ctypes.data))
        return k, v

    def step(self, t: int, kv_dtype: str = "f64"):
        """(true_q [L][hq][d] f32, approx_q, new_k [L][hkv][d], new_v); rows None at t = 0."""
        s = self.shape
        code, npdt = _DT[kv_dtype]
        tq = np.empty((s.num_layers, s.num_q_heads, s.head_dim), np.float32)
        aq = np.empty_like(tq)
        nk = nv = None
        if t >= 1:
            nk = np.empty((s.num_layers, s.num_kv_heads, s.head_dim), npdt)
            nv = np.empty_like(nk)
        check(self.lib.clo_trace_step(self.h, t, tq.ctypes.data, aq.ctypes.data,
                                      None if nk is None else nk.ctypes.data,
                                      None if nv is None else nv.ctypes.data, code))
        return tq, aq, nk, nv


class TraceSource:
    """StepSource over recorded traces (one per sequence of the batch).

    Arrays in the layout of workload.SyntheticWorkload:
      prompt_k/v [B][L][H][n_prompt][d]  storage dtype
      true_q/approx_q [steps+1][B][L][hq][d] float32
      new_k/v [steps][B][L][H][d]        storage dtype
    """

    alias_layers = False

    def __init__(self, paths, kv_dtype: str = "f32"):
        if isinstance(paths, (str, bytes)) or hasattr(paths, "__fspath__"):
            paths = [paths]
        traces = [Trace(p) for p in paths]
        t0 = traces[0]
        for t in traces[1:]:
            if (t.shape, t.n_prompt, t.n_steps) != (t0.shape, t0.n_prompt, t0.n_steps):
                raise _lib.ShapeError("ShapeError: batched traces must share shape, prompt and step counts")
        self.shape, self.n_prompt, self.steps = t0.shape, t0.n_prompt, t0.n_steps
        self.batch, self.kv_dtype = len(traces), kv_dtype
        self.element_width = t0.element_width
        L, HQ, H, d = self.shape.num_layers, self.shape.num_q_heads, self.shape.num_kv_heads, self.shape.head_dim
        npdt = _DT[kv_dtype][1]
        B, S, n = self.batch, self.steps, self.n_prompt
        self.prompt_k = np.empty((B, L, H, n, d), npdt)
        self.prompt_v = np.empty_like(self.prompt_k)
        self.true_q = np.empty((S + 1, B, L, HQ, d), np.float32)
        self.approx_q = np.empty_like(self.true_q)
        self.new_k = np.empty((S, B, L, H, d), npdt)
        self.new_v = np.empty_like(self.new_k)
        for b, tr in enumerate(traces):
            for l in range(L):
                for g in range(H):
                    self.prompt_k[b, l, g], self.prompt_v[b, l, g] = tr.prompt(l, g, kv_dtype)
            for t in range(S + 1):
                tq, aq, nk, nv = tr.step(t, kv_dtype)
                self.true_q[t, b], self.approx_q[t, b] = tq, aq
                if t >= 1:
                    self.new_k[t - 1, b], self.new_v[t - 1, b] = nk, nv
            tr.close()

    # kvsim::StepSource accessors (sequence 0 unless given)
    def prompt_tokens(self) -> int:
        return self.n_prompt

    def decode_steps(self) -> int:
        return self.steps

    def true_query(self, t, layer, q_head, seq=0):
        return self.true_q[t, seq, layer, q_head]

    def approx_query(self, t, layer, q_head, seq=0):
        return self.approx_q[t, seq, layer, q_head]

    def new_k_row(self, t, layer, kv_head, seq=0):
        if t < 1:
            raise _lib.ArgumentError("ArgumentError: new KV rows exist only for decode steps")
        return self.new_k[t - 1, seq, layer, kv_head]

    def new_v_row(self, t, layer, kv_head, seq=0):
        if t < 1:
            raise _lib.ArgumentError("ArgumentError: new KV rows exist only for decode steps")
        return self.new_v[t - 1, seq, layer, kv_head]

    def step_new_kv(self, t: int):
        """New K/V rows of decode step t (1-based) as [B][L][H][d] storage arrays."""
        return self.new_k[t - 1], self.new_v[t - 1]


def write_trace(path, shape: Shape, prompt_k, prompt_v, true_q, new_k, new_v, element_width: int = 8):
    """write_trace (trace_io.cpp:83-127) of one sequence: prompt_k/v [L][H][n][d],
    true_q [S+1][L][hq][d] (the hidden blocks), new_k/v [S][L][H][d] (float64)."""
    lib = _lib.load()
    arrs = [np.ascontiguousarray(a, np.float64) for a in (prompt_k, prompt_v, true_q, new_k, new_v)]
    n, S = arrs[0].shape[2], arrs[2].shape[0] - 1
    s = _lib.ModelShape(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, 2)
    check(lib.clo_trace_write(str(path).encode(), C.byref(s), n, S, element_width,
                              *[a.ctypes.data for a in arrs]))


def record_trace(source, path, seq: int = 0, element_width: int = 8):
    """record_trace (trace_io.cpp:185-228) of sequence `seq` of a workload with
    the SyntheticWorkload array layout (storage rows widened to double)."""
    from .workload import widen
    kvd = source.kv_dtype
    pk = widen(source.prompt_k[seq], kvd)
    pv = widen(source.prompt_v[seq], kvd)
    L = source.shape.num_layers
    if pk.shape[0] != L:  # layer-aliased store: every layer reads the same rows
        pk = np.broadcast_to(pk, (L,) + pk.shape[1:])
        pv = np.broadcast_to(pv, (L,) + pv.shape[1:])
    nk = np.stack([widen(source.step_new_kv(t)[0][seq], kvd) for t in range(1, source.steps + 1)]) \
        if source.steps else np.zeros((0, L, source.shape.num_kv_heads, source.shape.head_dim))
    nv = np.stack([widen(source.step_new_kv(t)[1][seq], kvd) for t in range(1, source.steps + 1)]) \
        if source.steps else np.zeros_like(nk)
    write_trace(path, source.shape, pk, pv, source.true_q[:, seq].astype(np.float64), nk, nv, element_width)
