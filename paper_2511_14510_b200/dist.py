"""Multi-GPU partitioning of the decode path.

Every hot-path operation is per (sequence, layer, KV head) with no cross-head
dependency (engine.cpp:260-409), so the path shards two ways:
  * by request: each rank serves its own sequences — pure replicas, no
    collective (weak scaling; `bench.py --gpus N`);
  * by KV head: each rank serves a contiguous block of KV heads with their m
    GQA query heads (`EngineConfig.kv_head_offset` keeps the per-head seeds
    and profiles of the global model); head outputs [B][L][hq/G][d] are then
    all-gathered into [B][L][hq][d] — the only exchange step.
torch.distributed is the plumbing (NCCL on GPUs, gloo in CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HeadShard:
    kv0: int      # first global KV head
    n_kv: int     # KV heads on this rank
    q0: int       # first global query head
    n_q: int      # query heads on this rank


def request_shard(batch_total: int, world: int, rank: int) -> tuple[int, int]:
    """(first sequence, count) of `rank`'s share; remainders go to the low ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(batch_total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def kv_head_shard(num_q_heads: int, num_kv_heads: int, world: int, rank: int) -> HeadShard:
    """Contiguous KV-head block of `rank`, with its GQA query heads (the q head
    h belongs to KV group h // m, matrix.hpp:53-54)."""
    if num_kv_heads % world:
        raise ValueError("num_kv_heads must be divisible by the number of ranks")
    m = num_q_heads // num_kv_heads
    n_kv = num_kv_heads // world
    kv0 = rank * n_kv
    return HeadShard(kv0, n_kv, kv0 * m, n_kv * m)


def allgather_heads(local, group=None):
    """[B][L][hq_local][d] on every rank -> [B][L][hq][d] (rank-major head blocks)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=2)


def attach_head_exchange(engine, rank: int, world: int, group=None) -> None:
    """Fused head-output all-gather (include/clo.h, exchange.cuh): every rank
    exports its engine's exchange handle, the handles travel over the host
    process group (torch.distributed plumbing: gloo or NCCL object
    all-gather), each engine maps its peers' buffers, then a barrier so no
    rank steps before every peer is attached. After this the attention
    epilogues store head outputs straight into the peers' memory; there is no
    per-step collective launch."""
    import torch.distributed as dist
    mine = engine.exchange_handle(rank, world)
    if world == 1:
        engine.attach_peers([mine])
        return
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    engine.attach_peers(handles)
    dist.barrier(group=group)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Device time of a multi-rank region = the slowest rank's."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
