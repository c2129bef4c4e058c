"""Trace wire format (§8f rank 2): libclo's reader/writer (csrc/trace.cpp,
paper_2511_14510_b200/trace.py) against the compiled reference's
read_trace / write_trace / record_trace / TraceSource (trace_io.cpp), on CPU.
Mirrors trace_io_test.cpp: f64 round trip bit for bit, f32 quantisation
through float, sidecar keys, replay accessors (approx = layer l-1 block), and
the reader's error behaviour."""
import json
import os

import numpy as np
import pytest

from oracle.bind import Reference
from paper_2511_14510_b200 import _lib
from paper_2511_14510_b200.trace import Trace, TraceSource, record_trace, write_trace
from paper_2511_14510_b200.workload import Shape, SyntheticWorkload

needs_ref = pytest.mark.skipif(not Reference.available(), reason="reference library not built")


def _ref_trace(tmp_path, width, name="ref.bin", **kw):
    p = tmp_path / name
    args = dict(L=2, hq=4, hkv=2, d=8, n_prompt=24, steps=5, d_model=32, seed=7, width=width)
    args.update(kw)
    Reference().record_synthetic_trace(p, **args)
    return p


@needs_ref
@pytest.mark.parametrize("width", [8, 4])
def test_reader_matches_reference_reader(tmp_path, width):
    p = _ref_trace(tmp_path, width)
    hdr, prompt, hidden, step = Reference().read_trace(p)
    tr = Trace(p)
    assert (tr.shape.num_layers, tr.shape.num_q_heads, tr.shape.num_kv_heads, tr.shape.head_dim) == tuple(hdr[:4])
    assert (tr.n_prompt, tr.n_steps, tr.element_width) == tuple(hdr[4:])
    L, hq, H, d = hdr[:4]
    for l in range(L):
        for g in range(H):
            k, v = tr.prompt(l, g, "f64")
            np.testing.assert_array_equal(k, prompt[l, g, 0])
            np.testing.assert_array_equal(v, prompt[l, g, 1])
    for t in range(hdr[5] + 1):
        tq, aq, nk, nv = tr.step(t, "f64")
        for l in range(L):
            np.testing.assert_array_equal(tq[l].reshape(-1), hidden[t, l].astype(np.float32))
            # TraceSource::approx_query: the layer l-1 block, layer 0 its own (trace_io.cpp:244-252)
            np.testing.assert_array_equal(aq[l].reshape(-1), hidden[t, max(l - 1, 0)].astype(np.float32))
            if t:
                np.testing.assert_array_equal(nk[l], step[t - 1, l, 0])
                np.testing.assert_array_equal(nv[l], step[t - 1, l, 1])


@needs_ref
def test_f32_trace_is_float_quantised(tmp_path):
    """trace_io_test.cpp:75-91: a width-4 trace holds float(x) for every x."""
    p64, p32 = _ref_trace(tmp_path, 8, "a.bin"), _ref_trace(tmp_path, 4, "b.bin")
    k64, _ = Trace(p64).prompt(0, 0, "f64")
    k32, _ = Trace(p32).prompt(0, 0, "f64")
    np.testing.assert_array_equal(k32, k64.astype(np.float32).astype(np.float64))


@needs_ref
@pytest.mark.parametrize("width", [8, 4])
def test_writer_round_trips_through_reference_reader(tmp_path, width):
    wl = SyntheticWorkload(Shape(3, 4, 2, 16), batch=2, n_prompt=40, steps=4, kv_dtype="f32", seed=3)
    p = tmp_path / "ours.bin"
    record_trace(wl, p, seq=1, element_width=width)
    hdr, prompt, hidden, step = Reference().read_trace(p)
    assert tuple(hdr) == (3, 4, 2, 16, 40, 4, width)
    np.testing.assert_array_equal(prompt[:, :, 0], wl.prompt_k[1].astype(np.float64))
    np.testing.assert_array_equal(prompt[:, :, 1], wl.prompt_v[1].astype(np.float64))
    np.testing.assert_array_equal(hidden.reshape(5, 3, 4, 16), wl.true_q[:, 1].astype(np.float64))
    np.testing.assert_array_equal(step[:, :, 0], wl.new_k[:, 1].astype(np.float64))
    side = json.load(open(str(p) + ".json"))
    assert side["format"] == "kvsim-trace" and side["layers"] == 3 and side["num_q_heads"] == 4
    assert side["num_kv_heads"] == 2 and side["head_dim"] == 16 and side["n_prompt"] == 40
    assert side["n_steps"] == 4 and side["element_width"] == width


def test_trace_source_replays_recorded_workload(tmp_path):
    """record -> TraceSource gives back the workload's arrays (f32 storage is
    exact through a width-4 trace); approx queries become the layer l-1 blocks."""
    wl = SyntheticWorkload(Shape(2, 4, 2, 8), batch=2, n_prompt=24, steps=3, kv_dtype="f32", seed=5)
    paths = []
    for b in range(2):
        paths.append(tmp_path / f"s{b}.bin")
        record_trace(wl, paths[-1], seq=b, element_width=4)
    src = TraceSource(paths, kv_dtype="f32")
    assert (src.batch, src.n_prompt, src.steps) == (2, 24, 3)
    np.testing.assert_array_equal(src.prompt_k, wl.prompt_k)
    np.testing.assert_array_equal(src.new_v, wl.new_v)
    np.testing.assert_array_equal(src.true_q, wl.true_q)
    np.testing.assert_array_equal(src.approx_q[:, :, 1], wl.true_q[:, :, 0])
    np.testing.assert_array_equal(src.approx_q[:, :, 0], wl.true_q[:, :, 0])
    with pytest.raises(_lib.ArgumentError):
        src.new_k_row(0, 0, 0)


def test_bf16_storage_rounds_to_nearest_even(tmp_path):
    wl = SyntheticWorkload(Shape(1, 2, 1, 8), batch=1, n_prompt=16, steps=1, kv_dtype="f32", seed=9)
    p = tmp_path / "t.bin"
    record_trace(wl, p, element_width=8)
    k, _ = Trace(p).prompt(0, 0, "bf16")
    x = wl.prompt_k[0, 0, 0].astype(np.float32)
    u = x.view(np.uint32)
    want = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    np.testing.assert_array_equal(k, want)


def test_reader_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTATRACE" + b"\0" * 64)
    with pytest.raises(_lib.IoError):
        Trace(bad)
    with pytest.raises(_lib.IoError):
        Trace(tmp_path / "missing.bin")
    wl = SyntheticWorkload(Shape(1, 2, 1, 8), batch=1, n_prompt=16, steps=2, kv_dtype="f32", seed=9)
    good = tmp_path / "good.bin"
    record_trace(wl, good, element_width=4)
    blob = good.read_bytes()
    (tmp_path / "trunc.bin").write_bytes(blob[:-5])
    with pytest.raises(_lib.IoError, match="truncated"):
        Trace(tmp_path / "trunc.bin")
    (tmp_path / "trail.bin").write_bytes(blob + b"\0")
    with pytest.raises(_lib.IoError, match="trailing"):
        Trace(tmp_path / "trail.bin")
    width = bytearray(blob)
    width[8 + 4 * 7: 8 + 4 * 8] = (3).to_bytes(4, "little")
    (tmp_path / "width.bin").write_bytes(bytes(width))
    with pytest.raises(_lib.IoError, match="element_width"):
        Trace(tmp_path / "width.bin")
    with pytest.raises(_lib.IndexError_):
        Trace(good).prompt(1, 0)
    with pytest.raises(_lib.ShapeError):
        other = tmp_path / "other.bin"
        record_trace(SyntheticWorkload(Shape(1, 2, 1, 8), batch=1, n_prompt=20, steps=2, kv_dtype="f32"), other)
        TraceSource([good, other])
    os.remove(good)
