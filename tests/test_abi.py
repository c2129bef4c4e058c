"""CPU checks of the C-ABI boundary: the library loads, exports exactly what
include/clo.h declares, and its host-side pure functions of the path
(threshold, partition plan, window indices, byte accounting) equal the
oracle. No CUDA calls."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2511_14510_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "clo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(clo_[a-z0-9_]+)\s*\(", src))
    return {n for n in names if not n.endswith("_t")}


def test_header_declares_the_binding_table():
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol(clo):
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in clo.clo_build_info()


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def _thr(clo, s, eta=0.8, p=3.0):
    v = C.c_double()
    _lib.check(clo.clo_compute_threshold(s, eta, p, C.byref(v)))
    return v.value


def test_threshold_equals_oracle(clo, oracle):
    for s in np.linspace(0, 1, 101):
        assert _thr(clo, s) == oracle.compute_threshold(s)
    assert _thr(clo, 0.5) == pytest.approx(-0.95164126255001177, abs=1e-15)  # head_profile_test.cpp:47-51
    with pytest.raises(_lib.ArgumentError):
        _thr(clo, 1.5)


def test_plan_partition_equals_oracle(clo, oracle):
    rng = np.random.default_rng(3)
    for _ in range(100):
        L, H = int(rng.integers(1, 6)), int(rng.integers(1, 9))
        diff = rng.uniform(-1, 1, (L, H))
        args = (float(rng.uniform(1e-6, 1e-3)), 2e10, float(rng.uniform(1e5, 1e7)), 1000,
                int(rng.choice([0, 0, H * 1000, H * 1000 + 3000])))
        out = np.zeros((L, H), np.int32)
        n_p, nd = C.c_int(), C.c_int()
        _lib.check(clo.clo_plan_partition(diff.ctypes.data, L, H, *args, out.ctypes.data, C.byref(n_p),
                                          C.byref(nd)))
        want, wn_p, wnd = oracle.plan_partition(diff, *args)
        assert np.array_equal(out.astype(bool), want) and n_p.value == wn_p and nd.value == wnd
    with pytest.raises(_lib.ConfigError):  # layer 0 cannot fit the budget
        d = np.zeros((2, 4))
        _lib.check(clo.clo_plan_partition(d.ctypes.data, 2, 4, 1e-3, 2e10, 2e6, 1000, 3000,
                                          np.zeros(8, np.int32).ctypes.data, C.byref(C.c_int()),
                                          C.byref(C.c_int())))


def test_window_indices_equal_oracle(clo, oracle):
    for n in (1, 2, 4, 10, 67, 68, 69, 100, 5000):
        for sink, recent in ((4, 64), (0, 64), (4, 0), (2, 8), (0, 0)):
            out = np.zeros(sink + recent + 1, np.int32)
            cnt, cl = C.c_int(), C.c_int()
            _lib.check(clo.clo_sink_recent_indices(n, sink, recent, out.ctypes.data, C.byref(cnt), C.byref(cl)))
            want, wcl = oracle.sink_recent_indices(n, sink, recent)
            assert list(out[: cnt.value]) == list(want) and bool(cl.value) == wcl


def test_cache_bytes_equal_oracle(clo, oracle):
    for args in ((1, 1000, 0, 0, 0, 128, 2), (248, 2048, 68, 32, 32, 128, 2), (0, 100, 68, 4, 8, 64, 2)):
        assert clo.clo_cache_bytes(*args) == oracle.cache_bytes(*args)


def test_config_defaults_mirror_engine_config(clo):
    c = _lib.EngineConfigC()
    clo.clo_engine_config_defaults(C.byref(c))
    # engine.hpp:30-49
    assert (c.sink_tokens, c.recent_tokens, c.hash_bits, c.retriever_seed, c.policy, c.retriever) == \
        (4, 64, 256, 1, _lib.POLICY_SIMILARITY, _lib.RETRIEVER_EXACT)


def test_engine_without_device_fails_loudly(clo):
    """No CPU fallback: on a box without a GPU engine creation is a CudaError."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    c = _lib.EngineConfigC()
    clo.clo_engine_config_defaults(C.byref(c))
    c.shape = _lib.ModelShape(2, 4, 2, 128, 2)
    c.k, c.n_prompt, c.max_steps = 8, 64, 4
    tau = np.zeros(4)
    qi = np.ones(8)
    pers = np.array([1, 1, 0, 0], np.int32)
    h = C.c_void_p()
    st = clo.clo_engine_create(C.byref(c), tau.ctypes.data, qi.ctypes.data, pers.ctypes.data, C.byref(h))
    assert st == 8  # CLO_ERR_CUDA


def test_cpp_shim_compiles_links_and_runs(tmp_path):
    """include/clo/kvsim.hpp: a kvsim-style C++ caller builds against the
    library and gets the reference's exception types (tests/cpp/shim_check.cpp)."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("no C++ compiler")
    exe = tmp_path / "shim_check"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_check.cpp"), "-L", libdir, "-lclo",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    try:
        import torch
        gpu = torch.cuda.is_available()
    except ImportError:
        gpu = False
    from paper_2511_14510_b200.trace import record_trace
    from paper_2511_14510_b200.workload import Shape, SyntheticWorkload
    trace = tmp_path / "t.bin"
    record_trace(SyntheticWorkload(Shape(2, 4, 2, 8), batch=1, n_prompt=16, steps=2, kv_dtype="f32"), trace)
    r = subprocess.run([str(exe), "gpu" if gpu else "cpu", str(trace)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)


@pytest.mark.gpu
def test_cpp_shim_decodes_on_gpu_like_the_python_path(tmp_path):
    """The kvsim-named C++ DecodeEngine (include/clo/kvsim.hpp, engine.hpp:91-139)
    drives prefill + decode_step on the GPU over a trace, and its
    cache_state_json equals the Python path's on the same inputs and config."""
    import json
    import subprocess
    import numpy as np
    from paper_2511_14510_b200 import DecodeEngine, EngineConfig, ModeFlags, ModelShape, PartitionPlan
    from paper_2511_14510_b200 import profiles_from_arrays
    from paper_2511_14510_b200.trace import TraceSource, record_trace
    from paper_2511_14510_b200.workload import Shape, SyntheticWorkload
    exe = tmp_path / "shim_check"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_check.cpp"), "-L", libdir, "-lclo",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    L, hq, hkv, d, n, steps = 3, 8, 2, 64, 300, 10
    trace = tmp_path / "t.bin"
    record_trace(SyntheticWorkload(Shape(L, hq, hkv, d), batch=1, n_prompt=n, steps=steps, kv_dtype="f32",
                                   sigma_step=0.15, seed=9), trace)
    out = tmp_path / "shim_state.json"
    r = subprocess.run([str(exe), "gpu", str(trace), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    shim_state = json.loads(out.read_text())
    m = hq // hkv
    tau = np.array([[0.55 + 0.1 * ((l + g) % 4) for g in range(hkv)] for l in range(L)])
    qimp = np.broadcast_to(1.0 + np.arange(m), (L, hkv, m)).copy()
    # the shim keeps EngineConfig's defaults (engine.hpp:30-49), compute_oracle_error included
    cfg = EngineConfig(shape=ModelShape(L, hq, hkv, d, 4), k=64, retriever="sign_hash", retriever_seed=5,
                       policy="similarity", mode=ModeFlags(), batch=1, kv_dtype="f32", compute_oracle_error=True)
    eng = DecodeEngine(cfg, profiles_from_arrays(tau, qimp), PartitionPlan(layers=[list(range(hkv))] + [[]] * (L - 1)),
                       TraceSource(trace, kv_dtype="f32"))
    eng.run()
    py_state = json.loads(eng.cache_state_json())
    assert shim_state["totals"]["misses"] > 0 and shim_state["totals"]["hits"] > 0
    assert shim_state["totals"]["mean_output_error"] > 0.0
    assert shim_state == py_state
