"""Fused head-output exchange of KV-head sharding (include/clo.h
clo_engine_exchange_handle / clo_engine_attach_peers, csrc/exchange.cuh) on
one B200: shard engines in one process (shared pointers) and in separate
processes (CUDA IPC mappings of the same device) each produce the WHOLE
model's outputs [B][L][hq][d], equal to the unsharded engine's — the
per-layer all-gather of SURVEY.md §8e without an NCCL launch. Selections and
decisions are bit-identical; outputs agree to float rounding (the tensor-core
kernel spreads a head's attend set over warps by the rank's own head count,
so the partial-merge order differs between shardings; every configuration is
bit-reproducible run to run, see test_outputs_bit_reproducible). The world-size
2 host plumbing (handle exchange over torch.distributed) runs here exactly as
it does across GPUs; only the peer mapping differs (same device vs NVLink)."""
import ctypes as C
import dataclasses
import os
import socket

import numpy as np
import pytest

from paper_2511_14510_b200 import DecodeEngine, PartitionPlan, _lib, profiles_from_arrays
from paper_2511_14510_b200.dist import kv_head_shard
from paper_2511_14510_b200.workload import HeadSlice
from tests.engine_harness import make_case

pytestmark = pytest.mark.gpu


def _case(hq=16, hkv=4, steps=5, batch=2):
    return make_case(L=3, hq=hq, hkv=hkv, d=128, n_prompt=600, steps=steps, k=64, batch=batch,
                     kv_dtype="bf16", sink=4, recent=64, seed=9)


def _unsharded(case):
    full = DecodeEngine(case["cfg"], profiles_from_arrays(case["tau"], case["qimp"]), case["plan"], case["wl"])
    full.run()
    want = np.stack(full.collected_outputs())  # [steps][B][L][hq][d]
    heads = {(l, g): full.head(l, g) for l in range(case["cfg"].shape.num_layers)
             for g in range(case["cfg"].shape.num_kv_heads)}
    full.close()
    return want, heads


def _shard_engine(case, world, rank):
    cfg, wl = case["cfg"], case["wl"]
    s = cfg.shape
    sh = kv_head_shard(s.num_q_heads, s.num_kv_heads, world, rank)
    sl = slice(sh.kv0, sh.kv0 + sh.n_kv)
    scfg = dataclasses.replace(cfg, shape=dataclasses.replace(s, num_q_heads=sh.n_q, num_kv_heads=sh.n_kv),
                               kv_head_offset=sh.kv0)
    plan = PartitionPlan(layers=[[g - sh.kv0 for g in heads if sh.kv0 <= g < sh.kv0 + sh.n_kv]
                                 for heads in case["plan"].layers])
    return DecodeEngine(scfg, profiles_from_arrays(case["tau"][:, sl], case["qimp"][:, sl]), plan,
                        HeadSlice(wl, sh.kv0, sh.n_kv, sh.q0, sh.n_q)), sh


def _attach_in_process(engines):
    world = len(engines)
    handles = [e.exchange_handle(r, world) for r, e in enumerate(engines)]
    for e in engines:
        e.attach_peers(handles)


def _step_all(engines, t):
    """One decode step of every shard, launched back to back with device
    resident inputs (no host sync in between: each step's finish kernel waits
    for the other shards' arrivals), then synchronised."""
    import torch
    lib = _lib.load()
    keep, outs = [], []
    # one stream per shard: graphs launched into the legacy default stream
    # would serialise, and shard 0's finish kernel would wait for shard 1's
    # arrivals forever (then time out)
    streams = getattr(_step_all, "streams", None)
    if streams is None or len(streams) < len(engines):
        streams = _step_all.streams = [torch.cuda.Stream() for _ in engines]
    ios = []
    for e in engines:  # inputs first: a device sync after a launch would wait on its finish kernel
        src = e.source
        nk, nv = src.step_new_kv(t)
        tq = torch.from_numpy(np.ascontiguousarray(src.true_q[t])).cuda()
        aq = torch.from_numpy(np.ascontiguousarray(src.approx_q[t])).cuda()
        dk = torch.from_numpy(np.ascontiguousarray(nk).view(np.int16)).cuda()
        dv = torch.from_numpy(np.ascontiguousarray(nv).view(np.int16)).cuda()
        s = e.cfg.shape
        out = torch.full((e.cfg.batch, s.num_layers, e.world * s.num_q_heads, s.head_dim), float("nan"),
                         device="cuda")
        keep.append((tq, aq, dk, dv))
        outs.append(out)
        ios.append(_lib.StepIO(tq.data_ptr(), aq.data_ptr(), dk.data_ptr(), dv.data_ptr(), out.data_ptr(), 0))
    torch.cuda.synchronize()
    for e, st, io in zip(engines, streams, ios):
        _lib.check(lib.clo_decode_step(e.h, C.byref(io), C.c_void_p(st.cuda_stream)))
    for e in engines:
        _lib.check(lib.clo_engine_synchronize(e.h))
        e.current_step = t
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("world", [2, 4])
def test_in_process_shards_all_gather(world):
    case = _case()
    want, heads = _unsharded(case)
    engines = [_shard_engine(case, world, r) for r in range(world)]
    eng = [e for e, _ in engines]
    _attach_in_process(eng)
    for e in eng:
        e.prefill()
    for t in range(1, case["wl"].steps + 1):
        outs = _step_all(eng, t)
        for r, out in enumerate(outs):
            assert np.isfinite(out).all(), f"rank {r} step {t}: exchange left holes"
            np.testing.assert_allclose(out, want[t - 1], rtol=1e-5, atol=1e-6, err_msg=f"rank {r} step {t}")
    for (e, sh) in engines:  # selections and decisions of every shard = the unsharded ones
        for l in range(case["cfg"].shape.num_layers):
            for g in range(sh.n_kv):
                a, b = e.head(l, g), heads[(l, sh.kv0 + g)]
                assert (a["hits"], a["misses"]) == (b["hits"], b["misses"])
                np.testing.assert_array_equal(a["entry_indices"], b["entry_indices"])
    for e in eng:
        e.close()


def test_lost_peer_reports_timeout(monkeypatch):
    """A shard whose peer stops stepping surfaces CLO_ERR_CUDA at the next
    synchronising call instead of hanging the GPU."""
    import subprocess
    import sys
    code = r"""
import ctypes as C, numpy as np, sys
sys.path.insert(0, %r)
from tests.test_gpu_exchange import _case, _shard_engine, _attach_in_process
from paper_2511_14510_b200 import _lib
case = _case(steps=2)
eng = [_shard_engine(case, 2, r)[0] for r in range(2)]
_attach_in_process(eng)
for e in eng:
    e.prefill()
try:
    eng[0].decode_step()   # rank 1 never steps
except _lib.CloError as ex:
    print("RAISED", type(ex).__name__, ex)
    sys.exit(0)
print("NO ERROR")
sys.exit(1)
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CLO_EXCHANGE_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "exchange timed out" in r.stdout


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2511_14510_b200.dist import attach_head_exchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = _case()
        e, _ = _shard_engine(case, world, rank)
        attach_head_exchange(e, rank, world)
        e.run()
        q.put((rank, np.stack(e.collected_outputs()), None))
        e.close()
    except Exception as ex:  # noqa: BLE001 - report to the parent
        q.put((rank, None, repr(ex)))
    finally:
        dist.destroy_process_group()


def test_two_processes_cuda_ipc_all_gather():
    """Two processes, one shard each, handles exchanged over gloo, peer
    buffers mapped with cudaIpcOpenMemHandle: the multi-process protocol
    bench.py --config 4 uses across GPUs."""
    import torch.multiprocessing as mp
    case = _case()
    want, _ = _unsharded(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, outs, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        got[rank] = outs
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(2):
        np.testing.assert_allclose(got[rank], want, rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(got[0], got[1])  # every rank holds the same gathered outputs


def test_outputs_bit_reproducible():
    """Two engines on the same inputs: bit-identical outputs (the partial
    merge order is fixed by the work decomposition, not by arrival order)."""
    case = _case(steps=3)
    a, _ = _unsharded(case)
    b, _ = _unsharded(case)
    np.testing.assert_array_equal(a, b)
