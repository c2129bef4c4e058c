"""World-size-2 checks of the multi-GPU partitioning logic on CPU (gloo):
KV-head sharding + head-output all-gather and request sharding reproduce the
unsharded decode step exactly (the per-rank compute here is the CPU oracle;
on GPUs the same shard plans drive the CUDA engine, see
tests/test_gpu_shard.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_14510_b200.dist import allgather_heads, kv_head_shard, max_over_ranks, request_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_case():
    from tests.engine_harness import make_case
    return make_case(L=2, hq=8, hkv=4, d=16, n_prompt=80, steps=4, k=8, batch=2, retriever="exact",
                     kv_dtype="f32", sigma_step=0.2)


def _run_oracle(case, b, heads=None):
    """Oracle decode of sequence b, restricted to KV heads [kv0, kv0+n_kv)."""
    from oracle.bind import Oracle
    from tests.engine_harness import oracle_cfg
    o = Oracle()
    wl = case["wl"]
    pk, pv, tq, aq, nk, nv = wl.oracle_inputs(b)
    c = oracle_cfg(case)
    tau, qimp, pers = case["tau"], case["qimp"], case["persistent"]
    if heads is not None:
        kv0, n_kv, q0, n_q = heads.kv0, heads.n_kv, heads.q0, heads.n_q
        c.num_kv_heads, c.num_q_heads = n_kv, n_q
        pk, pv = pk[:, kv0:kv0 + n_kv], pv[:, kv0:kv0 + n_kv]
        nk, nv = nk[:, :, kv0:kv0 + n_kv], nv[:, :, kv0:kv0 + n_kv]
        tq, aq = tq[:, :, q0:q0 + n_q], aq[:, :, q0:q0 + n_q]
        tau, qimp, pers = tau[:, kv0:kv0 + n_kv], qimp[:, kv0:kv0 + n_kv], pers[:, kv0:kv0 + n_kv]
    e = o.engine(c, np.ascontiguousarray(tau), np.ascontiguousarray(qimp), np.ascontiguousarray(pers),
                 np.ascontiguousarray(pk), np.ascontiguousarray(pv))
    e.prefill(np.ascontiguousarray(tq[0]))
    outs = []
    for t in range(1, wl.steps + 1):
        outs.append(e.decode_step(np.ascontiguousarray(tq[t]), np.ascontiguousarray(aq[t]),
                                  np.ascontiguousarray(nk[t - 1]), np.ascontiguousarray(nv[t - 1])))
    return np.stack(outs)  # [steps][L][hq_local][d]


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = _shard_case()
        s = case["cfg"].shape
        if mode == "heads":
            sh = kv_head_shard(s.num_q_heads, s.num_kv_heads, world, rank)
            mine = torch.from_numpy(np.stack([_run_oracle(case, b, sh) for b in range(case["wl"].batch)]))
            # [B][steps][L][hq_local][d] -> gather along the head axis (dim 3)
            full = allgather_heads(mine.permute(0, 1, 2, 3, 4).reshape(-1, s.num_layers, sh.n_q, s.head_dim))
            full = full.reshape(case["wl"].batch, case["wl"].steps, s.num_layers, s.num_q_heads, s.head_dim)
            result = full.numpy()
        else:
            start, cnt = request_shard(case["wl"].batch, world, rank)
            mine = [torch.from_numpy(_run_oracle(case, b)) for b in range(start, start + cnt)]
            parts = [None] * world
            dist.all_gather_object(parts, [(start + i, m.numpy()) for i, m in enumerate(mine)])
            result = dict(x for p in parts for x in p)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((result, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["heads", "requests"])
def test_two_rank_sharding_reproduces_unsharded_step(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    result, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0  # max over ranks
    case = _shard_case()
    for b in range(case["wl"].batch):
        want = _run_oracle(case, b)
        got = result[b]
        np.testing.assert_array_equal(got, want)


def test_shard_plans():
    assert [request_shard(16, 3, r) for r in range(3)] == [(0, 6), (6, 5), (11, 5)]
    sh = kv_head_shard(32, 8, 4, 2)
    assert (sh.kv0, sh.n_kv, sh.q0, sh.n_q) == (4, 2, 16, 8)
    with pytest.raises(ValueError):
        kv_head_shard(32, 8, 3, 0)


class _FakeEngine:
    """Stands in for DecodeEngine in the host half of the exchange protocol."""

    def __init__(self, rank):
        self.rank, self.attached = rank, None

    def exchange_handle(self, rank, world):
        assert rank == self.rank
        return bytes([rank]) * 256

    def attach_peers(self, handles):
        self.attached = list(handles)


def _exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_14510_b200.dist import attach_head_exchange
        e = _FakeEngine(rank)
        attach_head_exchange(e, rank, world)
        q.put((rank, e.attached))
    finally:
        dist.destroy_process_group()


def test_head_exchange_handles_travel_in_rank_order():
    """Host plumbing of the fused head-output all-gather (dist.attach_head_exchange):
    every rank ends up with all handles, in rank order, before anyone steps."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert got[r] == [bytes([0]) * 256, bytes([1]) * 256]
