"""ctypes binding of include/clo.h (paper_2511_14510_b200/libclo.so).

The library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2511_14510_b200/csrc`). Loading fails loudly when it is missing:
there is no CPU fallback for the CLO path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CLO_LIB") or os.path.join(HERE, "libclo.so")  # CLO_LIB: A/B builds

# clo_status (errors.hpp:10-41 taxonomy)
STATUS_NAMES = {
    0: "OK", 1: "ShapeError", 2: "ArgumentError", 3: "NumericError", 4: "IndexError",
    5: "ContractError", 6: "ConfigError", 7: "IoError", 8: "CudaError", 9: "InternalError",
}

RETRIEVER_EXACT, RETRIEVER_SIGN_HASH = 0, 1
POLICY_SIMILARITY, POLICY_LRU, POLICY_LFU, POLICY_PREFETCH_ONLY = 0, 1, 2, 3
DTYPE_BF16, DTYPE_F32, DTYPE_F64 = 0, 1, 2
SYNC_CPU_CENTRIC, SYNC_GPU_CENTRIC = 0, 1
HOST_HUGEPAGES = 1
EXCHANGE_HANDLE_BYTES = 256  # CLO_EXCHANGE_HANDLE_BYTES


class CloError(RuntimeError):
    """Base of the kvsim-style exception taxonomy (errors.hpp:10-41)."""

    code = 9


class ShapeError(CloError):
    code = 1


class ArgumentError(CloError):
    code = 2


class NumericError(CloError):
    code = 3


class IndexError_(CloError):  # noqa: N801 - kvsim::IndexError
    code = 4


class ContractError(CloError):
    code = 5


class ConfigError(CloError):
    code = 6


class IoError(CloError):
    code = 7


class CudaError(CloError):
    code = 8


_ERRORS = {c.code: c for c in (ShapeError, ArgumentError, NumericError, IndexError_, ContractError,
                               ConfigError, IoError, CudaError)}


class ModelShape(C.Structure):
    """matrix.hpp:46-66."""

    _fields_ = [("num_layers", C.c_int), ("num_q_heads", C.c_int), ("num_kv_heads", C.c_int),
                ("head_dim", C.c_int), ("bytes_per_element", C.c_int)]


class EngineConfigC(C.Structure):
    """clo_engine_config (engine.hpp:30-49 + B200 fields)."""

    _fields_ = [
        ("shape", ModelShape), ("k", C.c_int), ("sink_tokens", C.c_int), ("recent_tokens", C.c_int),
        ("retriever", C.c_int), ("hash_bits", C.c_int), ("retriever_seed", C.c_uint64),
        ("policy", C.c_int), ("always_miss", C.c_int), ("always_hit", C.c_int),
        ("has_tau_override", C.c_int), ("tau_override", C.c_double), ("sync_override", C.c_int),
        ("collect_outputs", C.c_int), ("compute_oracle_error", C.c_int), ("batch", C.c_int),
        ("n_prompt", C.c_int), ("max_steps", C.c_int), ("kv_dtype", C.c_int),
        ("kv_head_offset", C.c_int), ("device", C.c_int), ("victim_rows", C.c_int),
    ]


class StepIO(C.Structure):
    _fields_ = [("true_q", C.c_void_p), ("approx_q", C.c_void_p), ("new_k", C.c_void_p),
                ("new_v", C.c_void_p), ("out", C.c_void_p), ("on_host", C.c_int)]


class Metrics(C.Structure):
    _fields_ = [
        ("steps", C.c_uint64), ("hits", C.c_uint64), ("misses", C.c_uint64), ("lookups", C.c_uint64),
        ("hit_ratio", C.c_double), ("transferred_bytes", C.c_uint64),
        ("persistent_bytes", C.c_uint64), ("gathered_bytes_device", C.c_uint64),
        ("cache_bytes_current", C.c_uint64), ("host_bytes", C.c_uint64),
        ("device_persistent_bytes", C.c_uint64), ("sync_mode", C.c_int),
        ("mean_output_error", C.c_double),
    ]


class HeadState(C.Structure):
    _fields_ = [
        ("hits", C.c_uint64), ("misses", C.c_uint64), ("transferred_bytes", C.c_uint64),
        ("persistent_bytes", C.c_uint64), ("last_update_step", C.c_int),
        ("entry_last_update_step", C.c_int), ("labels_valid", C.c_int),
        ("window_held_tokens", C.c_int), ("placement", C.c_int), ("n_history", C.c_int),
    ]


class LayerTiming(C.Structure):  # clo_layer_timing (pipeline_sim.hpp:61-72 + wall_s)
    _fields_ = [("layer", C.c_int)] + [(f, C.c_double) for f in (
        "compute_s", "transfer_s", "hidden_s", "exposed_s", "mgmt_s", "sync_s", "retrieval_s", "total_s",
        "wall_s")]


class ProfilerConfig(C.Structure):  # clo_profiler_config
    _fields_ = [("blend_sequences", C.c_int), ("blend_steps", C.c_int), ("topk", C.c_int),
                ("sink_tokens", C.c_int), ("recent_tokens", C.c_int),
                ("eta", C.c_double), ("p", C.c_double), ("epsilon", C.c_double)]


class HeadProfileC(C.Structure):  # clo_head_profile
    _fields_ = [("q_importance", C.c_double * 16), ("kv_importance", C.c_double), ("s_hat", C.c_double),
                ("tau", C.c_double), ("difficulty", C.c_double), ("placement", C.c_int)]


class KernelSpan(C.Structure):  # clo_kernel_span
    _fields_ = [("name", C.c_char * 32), ("layer", C.c_int), ("start_ms", C.c_float), ("end_ms", C.c_float)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("layer", C.c_int), ("ms", C.c_float)]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_U64 = C.c_uint64
_D = C.c_double

# name -> (restype, argtypes): exactly the symbols include/clo.h declares.
SIGNATURES = {
    "clo_engine_config_defaults": (None, [C.POINTER(EngineConfigC)]),
    "clo_engine_create": (_I, [C.POINTER(EngineConfigC), _P, _P, _P, C.POINTER(_P)]),
    "clo_engine_destroy": (None, [_P]),
    "clo_engine_bind_host_kv": (_I, [_P, _P, _P, _I64, _I64, _I64]),
    "clo_engine_bind_host_kv_ex": (_I, [_P, _P, _P, _I64, _I64, _I64, _I64]),
    "clo_prefill": (_I, [_P, _P, _I, _P]),
    "clo_decode_step": (_I, [_P, C.POINTER(StepIO), _P]),
    "clo_engine_synchronize": (_I, [_P]),
    "clo_get_metrics": (_I, [_P, C.POINTER(Metrics)]),
    "clo_get_head_state": (_I, [_P, _I, _I, _I, C.POINTER(HeadState), _P, _P]),
    "clo_get_entry_rows": (_I, [_P, _I, _I, _I, _P, _P]),
    "clo_cache_state_json": (_I, [_P, _I, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "clo_engine_profile_step": (_I, [_P, C.POINTER(StepIO), _P, C.POINTER(KernelTime), _I, C.POINTER(_I)]),
    "clo_engine_timeline_step": (_I, [_P, C.POINTER(StepIO), _P]),
    "clo_get_timeline": (_I, [_P, C.POINTER(LayerTiming), _I, C.POINTER(LayerTiming), C.POINTER(_U64)]),
    "clo_timeline_spans": (_I, [_P, C.POINTER(KernelSpan), _I, C.POINTER(_I)]),
    "clo_timeline_json": (_I, [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "clo_engine_kernel_launches": (_U64, [_P]),
    "clo_engine_kernels_per_step": (_I, [_P]),
    "clo_engine_exchange_handle": (_I, [_P, _I, _I, _P]),
    "clo_engine_attach_peers": (_I, [_P, _P]),
    "clo_last_error": (C.c_char_p, []),
    "clo_host_alloc": (_I, [C.c_size_t, C.POINTER(_P)]),
    "clo_host_alloc_ex": (_I, [C.c_size_t, _I, C.POINTER(_P)]),
    "clo_host_alloc_numa": (_I, [C.c_size_t, _I, _I, C.POINTER(_P)]),
    "clo_device_numa_node": (_I, [_I, C.POINTER(_I)]),
    "clo_host_free": (_I, [_P]),
    "clo_host_register": (_I, [_P, C.c_size_t]),
    "clo_host_unregister": (_I, [_P]),
    "clo_sign_hash_projection": (_I, [_I, _I, _U64, _P]),
    "clo_encode_sign_hash": (_I, [_P, _I, _I64, _I, _I, _U64, _P, _P]),
    "clo_group_topk": (_I, [_P, _I, _I, _I, _P, _I, _P, _I, _U64, _I64, _I, _P, _P, _P]),
    "clo_topk_select_exact": (_I, [_P, _P, _I, _I64, _I, _I, _P, _P]),
    "clo_merge_group_topk": (_I, [_P, _I, _P, _P, _I, _P, _P]),
    "clo_lookup": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "clo_cosine_similarity": (_I, [_I, _I, _P, _P, _P, _P, _P]),
    "clo_aggregate_similarity": (_I, [_I, _I, _P, _P, _P, _P]),
    "clo_gather_rows": (_I, [_P, _I, _I, _I64, _P, _I, _P, _P]),
    "clo_gather_rows_ex": (_I, [_P, _I, _I, _I64, _P, _I, _P, _I, _I, _P, _P]),
    "clo_gather_rows_cpu_staged": (_I, [_P, _I, _I, _I64, _P, _I, _P, _P, _I, _P]),
    "clo_topk_attention": (_I, [_P, _I, _P, _P, _I, _I64, _I, _P, _I, _P, _P]),
    "clo_sink_recent_indices": (_I, [_I, _I, _I, _P, C.POINTER(_I), C.POINTER(_I)]),
    "clo_compute_threshold": (_I, [_D, _D, _D, C.POINTER(_D)]),
    "clo_compute_difficulty": (_I, [_D, _D, _D, C.POINTER(_D)]),
    "clo_plan_partition": (_I, [_P, _I, _I, _D, _D, _D, _U64, _U64, _P, C.POINTER(_I), C.POINTER(_I)]),
    "clo_cache_bytes": (_U64, [_I, _I, _I, _I, _I, _I, _I]),
    "clo_trace_open": (_I, [C.c_char_p, C.POINTER(_P)]),
    "clo_trace_close": (None, [_P]),
    "clo_trace_info": (_I, [_P, C.POINTER(ModelShape), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "clo_trace_prompt": (_I, [_P, _I, _I, _I, _P, _P]),
    "clo_trace_step": (_I, [_P, _I, _P, _P, _P, _P, _I]),
    "clo_trace_hidden": (_I, [_P, _I, _I, _P]),
    "clo_profiler_config_defaults": (None, [C.POINTER(ProfilerConfig)]),
    "clo_profile_heads": (_I, [_P, _I, C.POINTER(ProfilerConfig), _P, _P]),
    "clo_trace_write": (_I, [C.c_char_p, C.POINTER(ModelShape), _I, _I, _I, _P, _P, _P, _P, _P]),
    "clo_build_info": (C.c_char_p, []),
}

_lib = None


def load(path: str = LIB_PATH):
    """Loads libclo.so once; raises when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CLO path has no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status:
        msg = load().clo_last_error().decode()
        raise _ERRORS.get(status, CloError)(f"{STATUS_NAMES.get(status, status)}: {msg}")


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
