#!/usr/bin/env python3
"""Benchmark of the B200 CLO offloaded-KV decode step (BASELINE.json metric:
decode tokens/s @128K context; zero-copy PCIe GB/s vs link peak).

Workload = BASELINE.json configs[1]: Llama-3.1-8B attention shape (32 layers,
32 q / 8 kv heads, d=128), batch 16, 128K context, top-k 2048, head-wise
similarity cache + speculative prefetch, sign-hash (256-bit) retriever, bf16
KV in pinned host memory, layer 0 persistent (layer0_only_plan). A "step" is
one decode step: all 32 layers for all 16 sequences.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. Multi-GPU (torchrun): request sharding, each
rank serves its own 16 sequences with its own PCIe link (weak scaling, no
data-path collective); time = max over ranks.

Host-RAM note: 32 layers x 16 seqs x 8 heads x 128K x 2 (K,V) x 256 B = 256 GiB
would exceed the box's host RAM, so the synthetic host KV of the 32 layers is
ONE aliased buffer per (sequence, KV head) (layer_stride 0; new rows are
layer-invariant so aliasing stays consistent). Per-layer work is unchanged:
every layer has its own queries, codes, labels, cache slots and selections.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs, 1-based as in SURVEY.md §8d. configs[1] (= 2 here) is
# the headline the metric is quoted on and the default.
CONFIGS = {
    1: dict(name="configs[0]: single decode step, Llama-3-8B attention (32q/8kv, d128), batch 1, 32K ctx, "
                 "top-k 2048, cold gather of every offloaded head (always_miss)",
            layers=32, q_heads=32, kv_heads=8, head_dim=128, batch=1, ctx=32768, k=2048,
            always_miss=True, plan="layer0", shard="requests"),
    2: dict(name="configs[1]: Llama-3.1-8B attention shape (32 layers, 32q/8kv, d128), batch 16 per GPU, "
                 "128K ctx, top-k 2048, head-wise cache + prefetch, sign-hash 256b, layer 0 persistent",
            layers=32, q_heads=32, kv_heads=8, head_dim=128, batch=16, ctx=131072, k=2048,
            always_miss=False, plan="layer0", shard="requests"),
    3: dict(name="configs[2]: Qwen2.5-14B-Instruct-1M attention (48 layers, 40q/8kv, d128), batch 4, 512K ctx, "
                 "top-k 2048, persistent hard heads from plan_partition",
            layers=48, q_heads=40, kv_heads=8, head_dim=128, batch=4, ctx=524288, k=2048,
            always_miss=False, plan="partition", shard="requests"),
    4: dict(name="configs[3]: Llama-3.1-8B attention, 1M ctx, batch 8, KV heads sharded across GPUs "
                 "(per-GPU PCIe zero-copy, NCCL head-output all-gather)",
            layers=32, q_heads=32, kv_heads=8, head_dim=128, batch=8, ctx=1048576, k=2048,
            always_miss=False, plan="layer0", shard="heads"),
}
CONFIG2 = CONFIGS[2]
METRIC = "decode tokens/s @128K ctx (1/2/4/8 GPU); zero-copy PCIe GB/s vs link peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch")
    ap.add_argument("--ctx", type=int, default=0, help="override the config's context")
    ap.add_argument("--layers", type=int, default=0, help="override the config's layer count")
    ap.add_argument("--sigma", type=float, default=0.05, help="query drift per decode step")
    ap.add_argument("--sigma-layer", type=float, default=0.01)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--kv-layout", default="interleaved", choices=["split", "interleaved"],
                    help="host K/V layout: separate K and V matrices, or one token's K|V rows contiguous")
    ap.add_argument("--kv-dtype", default="bf16", choices=["bf16", "f32"],
                    help="storage type of the K/V rows (host store, cache slots, attention operands)")
    ap.add_argument("--victim-rows", type=int, default=-1,
                    help="HBM rows kept per offloaded head beyond its entry (-1: engine default 8k, 0: none)")
    ap.add_argument("--no-alias", action="store_true",
                    help="one host K/V region per layer (no layer aliasing): quantifies the aliased store's "
                         "effect on the gather; needs L times the host RAM (use --layers/--batch to fit)")
    ap.add_argument("--huge", action="store_true",
                    help="back the pinned host KV store with 2 MiB pages (GPU TLB reach for large stores)")
    ap.add_argument("--same-device", action="store_true",
                    help="testing only: every rank on cuda:0 with a gloo group (multi-rank functional check)")
    ap.add_argument("--allgather", default="fused", choices=["fused", "nccl"],
                    help="KV-head sharding exchange: fused into the attention epilogue over peer "
                         "memory (default), or an NCCL all_gather after each step (baseline)")
    args = ap.parse_args()
    args.cfg = dict(CONFIGS[args.config])
    args.batch = args.batch or args.cfg["batch"]
    args.ctx = args.ctx or args.cfg["ctx"]
    args.layers = args.layers or args.cfg["layers"]
    return args


# --------------------------------------------------------------------- helpers

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None
        self.window = None  # (t0, t1) of the timed region, time.monotonic()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def wait_first(self, timeout=3.0):
        """nvidia-smi needs ~0.1-0.3 s to its first sample: started before the
        warm-up, the sampler is live when the timed region begins."""
        end = time.monotonic() + timeout
        while self.proc and not self.rows and time.monotonic() < end:
            time.sleep(0.01)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        # samples inside the timed region; a region shorter than the 100 ms
        # sampling period (configs[0]: ~25 ms) takes the samples of the
        # warm-up + timed region instead and says so
        rows, window = [r for _, r in self.rows], "timed region"
        if self.window:
            inside = [r for t, r in self.rows if self.window[0] <= t <= self.window[1] + 0.05]
            if inside:
                rows = inside
            else:
                window = "warm-up + timed region (timed region shorter than the 100 ms sampling period)"
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4)
                          if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "window": window}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def head_profiles(args, threshold, plan_partition):
    """Synthetic head profiles and the persistent-head plan of the workload,
    identical in both arms. threshold(s, eta, p) = compute_threshold
    (head_profile.cpp:17-25); plan_partition(diff, t_comp_s, pcie_bw,
    mem_head_bytes, persist_bytes_per_head, hbm_budget_bytes) -> (persistent
    [L][H], n_p, dropped) (head_profile.cpp:80-154). Returns tau [L][H],
    q_importance [L][H][m], persistent [L][H] int32 and a one-line plan note."""
    from paper_2511_14510_b200.workload import Shape, synthetic_profiles
    C2 = args.cfg
    L, HQ, H, d, n, k, B = (args.layers, C2["q_heads"], C2["kv_heads"], C2["head_dim"], args.ctx, C2["k"],
                            args.batch)
    tau, qimp = synthetic_profiles(Shape(L, HQ, H, d), seed=args.seed, threshold=threshold)
    persistent = np.zeros((L, H), np.int32)
    persistent[0] = 1  # layer0_only_plan (engine.cpp:548-555)
    plan_info = "layer0_only_plan"
    if C2["plan"] == "partition":
        # plan_partition over synthetic profiles: difficulty = tau - (s_hat - eps),
        # eps = 0.05 (compute_difficulty :27-30), s_hat ~ U(0.5, 1) per head; N_p
        # from a 50 us compute window at the measured-order PCIe bandwidth; HBM
        # budget 80 GiB for the persistent KV of all `B` sequences.
        rs = np.random.default_rng(args.seed + 17)
        s_hat = rs.uniform(0.5, 1.0, (L, H))
        diff = tau - (s_hat - 0.05)
        row = 2 * d * 2
        pers, n_p, nd = plan_partition(diff, 5e-5, 5.0e10, float(2 * k * d * 2), row * (n + 4096) * B,
                                       80 * (1 << 30))
        persistent = np.asarray(pers, np.int32)
        plan_info = f"plan_partition: N_p={n_p}, persistent heads={int(persistent.sum())}/{L * H}, dropped={nd}"
    return tau, qimp, persistent, plan_info


def workload_config(args, plan_info, world):
    """The `config` object of the JSON line, identical in both arms."""
    C2 = args.cfg
    shard_heads = C2["shard"] == "heads" and world > 1
    return {"workload": C2["name"], "batch_per_gpu": args.batch, "ctx": args.ctx, "layers": args.layers,
            "k": C2["k"], "plan": plan_info,
            "parallelism": (f"kv-head-sharded x{world} (+{'fused P2P' if args.allgather == 'fused' else 'NCCL'} "
                            f"head-output all-gather)" if shard_heads else f"request-sharded x{world}"),
            "l2": "per-step working set (codes, slots, persistent KV) >> 126 MB L2",
            "host_kv": ("pinned, one buffer per (seq, layer, kv head), not aliased, "
                        if getattr(args, "no_alias", False) else
                        "pinned, one buffer per (seq, kv head) aliased across layers, ")
                       + ("K|V rows of a token contiguous (row stride 2d)" if args.kv_layout == "interleaved"
                          else "separate K and V matrices"),
            "kv_dtype": args.kv_dtype, "sigma_step": args.sigma, "sigma_layer": args.sigma_layer,
            "victim_rows": args.victim_rows if args.victim_rows >= 0 else "auto (8k, HBM-capped)"}


# ------------------------------------------------------------ reference arm

def reference_sample(args, steps: int, warmup: int, threads: int):
    """Times the reference's own DecodeEngine (oracle/_ref, compiled from
    /root/reference) on `threads` host threads, each one (sequence, layer, KV
    head) unit of the same workload at full context, the way the reference
    runner runs independent engines on a std::thread pool. Falls back to the
    C restatement ('port') when the reference library is absent."""
    from oracle.bind import EngineCfg, Oracle, Reference
    from paper_2511_14510_b200.workload import _normalize
    C2 = args.cfg
    d, m, n = C2["head_dim"], C2["q_heads"] // C2["kv_heads"], args.ctx
    rng = np.random.default_rng(args.seed)
    bf = lambda a: ((a.astype(np.float32).view(np.uint32) + 0x8000) & 0xFFFF0000).view(np.float32)
    pk = bf(rng.standard_normal((1, 1, n, d), np.float32)).astype(np.float64)
    pv = bf(rng.standard_normal((1, 1, n, d), np.float32)).astype(np.float64)
    q = _normalize(rng.standard_normal((1, m, d)))
    tq = np.empty((steps + 1, 1, m, d))
    aq = np.empty_like(tq)
    for t in range(steps + 1):
        if t:
            q = _normalize(q + args.sigma * rng.standard_normal(q.shape))
        tq[t] = q.astype(np.float32)
        aq[t] = _normalize(q + args.sigma_layer * rng.standard_normal(q.shape)).astype(np.float32)
    nk = bf(rng.standard_normal((steps, 1, 1, d), np.float32)).astype(np.float64)
    nv = bf(rng.standard_normal((steps, 1, 1, d), np.float32)).astype(np.float64)
    c = EngineCfg()
    c.num_layers, c.num_q_heads, c.num_kv_heads, c.head_dim, c.bytes_per_element = 1, m, 1, d, 2
    c.k, c.sink_tokens, c.recent_tokens = C2["k"], 4, 64
    c.always_miss = int(C2["always_miss"])
    c.retriever, c.hash_bits, c.retriever_seed, c.policy = 1, 256, 1, 0
    c.n_prompt, c.steps = n, steps
    if Reference.available():
        kind, lib = "reference", Reference()
    else:
        kind, lib = "port", None
    # the same head profiles and plan as our arm; thread w serves the w-th of
    # `threads` offloaded (layer, kv head) units spread evenly over the model
    prof_lib = lib or Oracle()
    tau_all, qimp_all, pers, _ = head_profiles(args, prof_lib.compute_threshold, prof_lib.plan_partition)
    offl = [(l, g) for l in range(pers.shape[0]) for g in range(pers.shape[1]) if not pers[l, g]]
    pick = [offl[int(i)] for i in np.linspace(0, len(offl) - 1, threads)] if offl else [(0, 0)] * threads
    tau = np.array([tau_all[l, g] for l, g in pick])
    qimp = np.array([qimp_all[l, g] for l, g in pick])
    t0 = time.time()
    if lib is not None:
        sps, pre = lib.bench_units(c, tau, qimp, pk, pv, tq, aq, nk, nv, threads, warmup)
        per_unit = float(np.mean(sps))
    else:  # C restatement, one unit per thread is not exposed: time one unit serially
        o = Oracle()
        e = o.engine(c, tau[:1].reshape(1, 1), qimp[:1].reshape(1, 1, m), np.zeros((1, 1), np.int32), pk, pv)
        e.prefill(tq[0])
        for t in range(1, warmup + 1):
            e.decode_step(tq[t], aq[t], nk[t - 1], nv[t - 1])
        ts = time.perf_counter()
        for t in range(warmup + 1, steps + 1):
            e.decode_step(tq[t], aq[t], nk[t - 1], nv[t - 1])
        per_unit = (time.perf_counter() - ts) / max(1, steps - warmup)
        threads = 1
    wall = time.time() - t0
    units_per_token_step = args.batch * args.layers * C2["kv_heads"]
    # `threads` units run concurrently; one decode step of the whole batch needs
    # units_per_token_step units, producing `batch` tokens.
    tokens_per_s = args.batch * threads / (units_per_token_step * per_unit)
    sample = (f"{threads} concurrent reference DecodeEngines, each one (sequence, layer, KV head) "
              f"unit at ctx={n}, m={m}, k={C2['k']}, sign-hash, similarity policy"
              f"{' (always_miss)' if C2['always_miss'] else ''}, head profiles (tau, q_importance) of "
              f"{threads} offloaded (layer, kv head) pairs of the same synthetic profile as the GPU arm, "
              f"{steps - warmup} timed decode_steps after {warmup} warm-up; {per_unit * 1e3:.1f} ms "
              f"per unit-step (mean over threads); wall {wall:.1f}s")
    extrap = (f"EXTRAPOLATED: tokens/s = B * threads / (units per batch step * mean unit-step time) with "
              f"{units_per_token_step} units per batch step (B={args.batch}, L={args.layers}, H={C2['kv_heads']}); "
              f"the full batch step is not run on the CPU (it would take "
              f"{units_per_token_step * per_unit / threads:.0f} s per step)")
    return {"value": tokens_per_s, "unit": "tokens/s", "cores": threads, "kind": kind, "sample": sample,
            "extrapolation": extrap, "cpu_model": cpu_model(), "sec_per_unit_step": per_unit}


def cpu_threads(args):
    """All host threads, capped so the per-thread reference engines (about four
    n x d double matrices each) stay within half of the host RAM."""
    threads = args.cpu_threads or os.cpu_count() or 1
    try:
        import psutil
        ram = psutil.virtual_memory().total
    except ImportError:
        ram = 64 << 30
    per_thread = 4 * args.ctx * args.cfg["head_dim"] * 8 + (1 << 28)
    return max(1, min(threads, int(0.5 * ram // per_thread)))


def _plan_info_reference(args):
    from oracle.bind import Oracle, Reference
    lib = Reference() if Reference.available() else Oracle()
    return head_profiles(args, lib.compute_threshold, lib.plan_partition)[3]


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = cpu_threads(args)
    # W warm-up and K timed decode steps of one (sequence, layer, KV head) unit
    # per host thread: a bounded sample of the batch step (~0.15 s per unit-step
    # at 128K, ~1.2 s at 1M)
    cb = reference_sample(args, args.warmup + args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * args.batch / cb["value"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, _plan_info_reference(args), args.gpus),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "extrapolation",
                                            "cpu_model")},
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- our arm

def run_ours(args):
    import torch

    world, rank, local = dist_env()
    if args.same_device:  # functional multi-rank check on a 1-GPU box (not a bench number)
        local = 0
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    elif world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPUs "
                         "(--same-device runs every rank on cuda:0 as a functional check)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.same_device:  # NCCL refuses two ranks on one device; gloo carries the host plumbing
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_14510_b200 import _lib
    from paper_2511_14510_b200.engine import (DecodeEngine, EngineConfig, HostKV, ModelShape, ModeFlags,
                                              layer0_only_plan, profiles_from_arrays)
    lib = _lib.load()
    C2 = args.cfg
    B, L, HQ_all, H_all, d, n, k = (args.batch, args.layers, C2["q_heads"], C2["kv_heads"],
                                    C2["head_dim"], args.ctx, C2["k"])
    # KV-head sharding (configs[3]): this rank serves a contiguous block of KV
    # heads for every sequence; request sharding: all heads of its own sequences.
    shard_heads = C2["shard"] == "heads" and world > 1
    from paper_2511_14510_b200.dist import kv_head_shard
    hs = kv_head_shard(HQ_all, H_all, world if shard_heads else 1, rank if shard_heads else 0)
    HQ, H = hs.n_q, hs.n_kv
    W, K = args.warmup, args.steps
    P = 2                       # profiled (instrumented-graph) steps
    TL = 4                      # timeline steps (measured LayerTiming breakdown)
    E = 0 if args.no_e2e else K  # end-to-end (host buffers) steps
    S = W + K + P + TL + E + (W if E else 0)
    nmax = n + S
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed * 1000 + rank)
    t_setup = time.time()

    # NUMA placement: this rank's pinned host shard lives on the
    # host node of its GPU's PCIe root, and its host threads run there, so the
    # zero-copy gathers never cross the socket interconnect.
    from paper_2511_14510_b200.engine import device_numa_node, numa_node_cpus
    node = device_numa_node(local)
    multi_node = os.path.exists("/sys/devices/system/node/node1")
    numa = {"gpu_node": node, "host_nodes": "multi" if multi_node else "single", "bound": False}
    if node >= 0 and multi_node:
        cpus = numa_node_cpus(node)
        if cpus:
            os.sched_setaffinity(0, cpus)
            numa["cpus"] = len(cpus)
        numa["bound"] = True

    # host KV: one aliased [B][1][H][nmax][d] bf16 buffer pair (see module doc)
    kvd = args.kv_dtype
    tdt = torch.bfloat16 if kvd == "bf16" else torch.float32
    esz = 2 if kvd == "bf16" else 4
    Lk = L if args.no_alias else 1
    hkv = HostKV(B, Lk, H, nmax, d, kvd, hugepages=args.huge, interleaved=args.kv_layout == "interleaved",
                 numa_node=node if numa["bound"] else -1)
    for b in range(B):
        for lk in range(Lk):
            for arr in (hkv.k, hkv.v):
                x = torch.randn((H, n, d), generator=gen, device=dev, dtype=torch.float32).to(tdt)
                for h in range(H):  # contiguous [n][d] block of pinned memory: direct D2H
                    if kvd == "bf16":
                        torch.from_numpy(arr[b, lk, h, :n].view(np.int16)).copy_(x[h].view(torch.int16))
                    else:
                        torch.from_numpy(arr[b, lk, h, :n]).copy_(x[h])

    # per-step inputs (device resident): drift-walk queries, layer-invariant new rows
    def norm(x):
        return x / x.norm(dim=-1, keepdim=True)
    tq = torch.empty((S + 1, B, L, HQ, d), device=dev)
    aq = torch.empty_like(tq)
    q = norm(torch.randn((B, L, HQ, d), generator=gen, device=dev))
    for t in range(S + 1):
        if t:
            q = norm(q + args.sigma * torch.randn(q.shape, generator=gen, device=dev))
        tq[t] = q
        aq[t] = norm(q + args.sigma_layer * torch.randn(q.shape, generator=gen, device=dev))
    nk = torch.randn((S, B, Lk, H, d), generator=gen, device=dev).to(tdt).expand(S, B, L, H, d).contiguous()
    nv = torch.randn((S, B, Lk, H, d), generator=gen, device=dev).to(tdt).expand(S, B, L, H, d).contiguous()
    fused_x = shard_heads and args.allgather == "fused"
    HQo = HQ * world if fused_x else HQ  # out's head extent
    out = torch.empty((B, L, HQo, d), device=dev)

    def thr(s, eta, p):
        v = C.c_double()
        _lib.check(lib.clo_compute_threshold(s, eta, p, C.byref(v)))
        return v.value

    def plan_partition(diff, t_comp_s, pcie_bw, mem_head_bytes, persist_bytes, budget):
        Lp, Hp = diff.shape
        pers = np.zeros((Lp, Hp), np.int32)
        n_p, nd = C.c_int(), C.c_int()
        _lib.check(lib.clo_plan_partition(np.ascontiguousarray(diff).ctypes.data, Lp, Hp, t_comp_s, pcie_bw,
                                          mem_head_bytes, persist_bytes, budget, pers.ctypes.data, C.byref(n_p),
                                          C.byref(nd)))
        return pers, n_p.value, nd.value
    tau, qimp, persistent, plan_info = head_profiles(args, thr, plan_partition)
    sl = slice(hs.kv0, hs.kv0 + hs.n_kv)
    tau, qimp, persistent = tau[:, sl].copy(), qimp[:, sl].copy(), persistent[:, sl].copy()

    class _Src:  # StepSource shape for DecodeEngine's constructor (prompt already in hkv)
        n_prompt, steps, alias_layers = n, S, not args.no_alias
        prompt_k = prompt_v = None

    cfg = EngineConfig(shape=ModelShape(L, HQ, H, d, esz), k=k, sink_tokens=4, recent_tokens=64,
                       retriever="sign_hash", hash_bits=256, retriever_seed=1, policy="similarity",
                       mode=ModeFlags(always_miss=C2["always_miss"]), batch=B, kv_dtype=kvd,
                       kv_head_offset=hs.kv0, device=local, victim_rows=args.victim_rows)
    from paper_2511_14510_b200.engine import PartitionPlan
    plan = PartitionPlan(layers=[[g for g in range(H) if persistent[l, g]] for l in range(L)])
    eng = DecodeEngine(cfg, profiles_from_arrays(tau, qimp), plan, _Src, host_kv=hkv)
    if fused_x:  # head outputs travel inside the attention epilogue (exchange.cuh)
        from paper_2511_14510_b200.dist import attach_head_exchange
        attach_head_exchange(eng, rank, world)
    t_pre = time.time()
    _lib.check(lib.clo_prefill(eng.h, tq[0].data_ptr(), 0, None))
    prefill_s = time.time() - t_pre
    setup_s = time.time() - t_setup

    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    t_idx = [0]

    def dev_io(t):
        return _lib.StepIO(tq[t].data_ptr(), aq[t].data_ptr(), nk[t - 1].data_ptr(), nv[t - 1].data_ptr(),
                           out.data_ptr(), 0)

    gathered_out = torch.empty((world, B, L, HQ, d), device=dev) if shard_heads else None

    def step_dev():
        t_idx[0] += 1
        io = dev_io(t_idx[0])
        _lib.check(lib.clo_decode_step(eng.h, C.byref(io), C.c_void_p(sp)))
        if shard_heads and not fused_x:  # baseline exchange: NCCL all-gather after the step
            dist.all_gather(list(gathered_out.unbind(0)), out)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if dist is None:
            return x
        tt = torch.tensor([x], device="cpu" if args.same_device else dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # ---- warm-up + timed region (inputs resident in HBM) -------------------
    clocks = ClockSampler(local).__enter__()  # live (first sample in) before the timed region
    clocks.wait_first()
    for _ in range(W):
        step_dev()
    m0 = eng.metrics()
    launches0 = eng.kernel_launches()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    t_region0 = time.monotonic()
    ev0.record(stream)
    for i in range(K):
        step_dev()
        step_ev[i].record(stream)
    ev1.record(stream)
    barrier()
    clocks.window = (t_region0, time.monotonic())
    clocks.__exit__(None, None, None)
    step_ms = [ev0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i]) for i in range(1, K)]
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = eng.kernel_launches() - launches0
    m1 = eng.metrics()
    ms_per_step = ms / K
    value = (1 if shard_heads else world) * B * K / (ms / 1e3)
    hits = m1["hits"] - m0["hits"]
    misses = m1["misses"] - m0["misses"]
    gathered = m1["gathered_bytes_device"] - m0["gathered_bytes_device"]

    # ---- instrumented steps: per-kernel device time inside the graph -------
    recs = (_lib.KernelTime * 4096)()
    cnt = C.c_int()
    per_kernel = {}
    pm0 = eng.metrics()
    for _ in range(P):
        t_idx[0] += 1
        io = dev_io(t_idx[0])
        _lib.check(lib.clo_engine_profile_step(eng.h, C.byref(io), C.c_void_p(sp), recs, 4096, C.byref(cnt)))
        for i in range(min(cnt.value, 4096)):
            r = recs[i]
            e = per_kernel.setdefault(r.name.decode(), {"ms": 0.0, "launches": 0})
            e["ms"] += r.ms
            e["launches"] += 1
    pm1 = eng.metrics()
    for e in per_kernel.values():
        e["ms"] /= P
        e["launches"] //= P
    prof_gathered = (pm1["gathered_bytes_device"] - pm0["gathered_bytes_device"]) / P
    prof_misses = (pm1["misses"] - pm0["misses"]) / P

    # ---- measured LayerTiming breakdown (the reference's categories) --------
    for _ in range(TL):
        t_idx[0] += 1
        io = dev_io(t_idx[0])
        _lib.check(lib.clo_engine_timeline_step(eng.h, C.byref(io), C.c_void_p(sp)))
    tl = eng.timeline()
    tt = tl["totals"]
    if os.environ.get("CLO_BENCH_SPANS"):  # Gantt dump of the last timeline step
        with open(os.environ["CLO_BENCH_SPANS"], "w") as f:
            json.dump(eng.timeline_spans(), f)
    n_tl = max(1, tl["steps"])
    layer_timing = {
        "steps": tl["steps"],
        "per_step_ms": {k[:-2]: round(1e3 * tt[k] / n_tl, 4) for k in
                        ("compute_s", "transfer_s", "hidden_s", "exposed_s", "mgmt_s", "sync_s", "retrieval_s",
                         "total_s", "wall_s")},
        "share_of_total": {k[:-2]: round(tt[k] / tt["total_s"], 4) if tt["total_s"] else None for k in
                           ("compute_s", "exposed_s", "mgmt_s", "sync_s", "retrieval_s")},
        "note": "pipeline_sim.hpp LayerTiming categories measured with CUDA events in the production stream "
                "layout; total = compute + exposed + mgmt + sync + retrieval (the reference's formula), "
                "wall = measured compute-stream time",
    }

    # ---- end-to-end through the C-ABI with pinned HOST buffers -------------
    e2e = None
    if E:
        h_tq = torch.empty((E + W, B, L, HQ, d), pin_memory=True)
        h_aq = torch.empty_like(h_tq, pin_memory=True)
        h_nk = torch.empty((E + W, B, L, H, d), dtype=tdt, pin_memory=True)
        h_nv = torch.empty_like(h_nk, pin_memory=True)
        h_out = torch.empty((B, L, HQo, d), pin_memory=True)
        base = t_idx[0]
        h_tq.copy_(tq[base + 1: base + 1 + E + W])
        h_aq.copy_(aq[base + 1: base + 1 + E + W])
        h_nk.copy_(nk[base: base + E + W])
        h_nv.copy_(nv[base: base + E + W])

        def step_host(i):
            t_idx[0] += 1
            io = _lib.StepIO(h_tq[i].data_ptr(), h_aq[i].data_ptr(), h_nk[i].data_ptr(), h_nv[i].data_ptr(),
                             h_out.data_ptr(), 1)
            _lib.check(lib.clo_decode_step(eng.h, C.byref(io), C.c_void_p(sp)))
        for i in range(W):
            step_host(i)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(W, W + E):
            step_host(i)
        e1.record(stream)
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1))
        h2d = (2 * B * L * HQ * d * 4) + 2 * B * L * H * d * esz
        d2h = B * L * HQo * d * 4
        e2e = {"value": (1 if shard_heads else world) * B * E / (ems / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / E}

    # ---- PCIe link peak (pinned cudaMemcpy H2D, 1 GiB, best of 5) ----------
    pin = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(6):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dbuf.copy_(pin, non_blocking=True)
        b_.record(stream)
        torch.cuda.synchronize(dev)
        best = max(best, (1 << 30) / (a.elapsed_time(b_) * 1e-3) / 1e9)
    del pin, dbuf

    # ---- roofline of the dominant kernel ------------------------------------
    peaks, peak_kind = measured_peaks()
    total_prof = sum(e["ms"] for e in per_kernel.values()) or 1.0
    dom = max(per_kernel, key=lambda kk: per_kernel[kk]["ms"]) if per_kernel else None
    row_b = d * esz
    W_ = 68
    attn_bytes_launch = B * H * 2 * (k + W_) * row_b          # K+V rows of k + window per head
    gather_ms = per_kernel.get("gather_zero_copy", {}).get("ms", 0.0)
    attn_ms = per_kernel.get("attention", {}).get("ms", 0.0)
    attn_launches = max(1, per_kernel.get("attention", {}).get("launches", 1))
    gather_gbs = prof_gathered / (gather_ms * 1e-3) / 1e9 if gather_ms else 0.0
    attn_gbs = attn_bytes_launch / ((attn_ms / attn_launches) * 1e-3) / 1e9 if attn_ms else 0.0
    sel_ms = per_kernel.get("select_offloaded", {}).get("ms", 0.0) + per_kernel.get("select_persistent", {}).get("ms", 0.0)
    sel_bytes = (prof_misses + B * H) * (n + (t_idx[0])) * (32 + 4)  # codes + u16 key write/read per scored key
    sel_gbs = sel_bytes / (sel_ms * 1e-3) / 1e9 if sel_ms else 0.0
    rooflines = {
        "gather_zero_copy": {"bound": "pcie", "achieved": gather_gbs, "peak": best, "unit": "GB/s",
                             "frac": gather_gbs / best if best else None,
                             "frac_of_gen5_x16_theoretical": gather_gbs / 64.0,
                             "traffic": None, "share": gather_ms / total_prof,
                             "bytes_per_unit": "2*k*d*e per missed (seq,layer,kv head) = 1 MiB"},
        "attention": {"bound": "hbm", "achieved": attn_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                      "frac": attn_gbs / peaks["hbm_gbs"], "traffic": None, "share": attn_ms / total_prof,
                      "bytes_per_unit": "2*(k+68)*d*e per (seq,kv head) per layer = 1.03 MiB"},
        "select": {"bound": "hbm", "achieved": sel_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                   "frac": sel_gbs / peaks["hbm_gbs"], "traffic": None, "share": sel_ms / total_prof,
                   "bytes_per_unit": "36 B per scored key (32 B code + u16 key write+read)"},
    }
    # measured traffic / algorithmic bytes from the committed ncu captures,
    # scaled to this run's per-launch algorithmic bytes (profiles/r1_traffic.json)
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            tr = json.load(f)
        launches_of = {"gather_zero_copy": per_kernel.get("gather_zero_copy", {}).get("launches", 1),
                       "attention": attn_launches,
                       "select": per_kernel.get("select_offloaded", {}).get("launches", 1)}
        alg_per_launch = {"gather_zero_copy": prof_gathered / max(1, launches_of["gather_zero_copy"]),
                          "attention": attn_bytes_launch,
                          "select": sel_bytes / max(1, launches_of["select"])}
        for kname, rl in rooflines.items():
            t = tr.get(kname)
            if not t:
                continue
            moved = t.get("pcie_read_bytes", 0) + t.get("dram_read_bytes", 0) + t.get("dram_write_bytes", 0) \
                if kname != "gather_zero_copy" else t["pcie_read_bytes"]
            ratio = moved / t["algorithmic_bytes"]
            rl["traffic"] = ratio * alg_per_launch[kname]
            rl["traffic_ratio"] = round(ratio, 4)
            rl["traffic_source"] = "profiles/r1_traffic.json: " + t["capture"]
    except (OSError, KeyError, ValueError):
        pass
    dom_name = "gather_zero_copy" if dom == "gather_zero_copy" else (
        "attention" if dom == "attention" else ("select" if dom and dom.startswith("select") else dom))
    roof = dict(rooflines.get(dom_name, rooflines["attention"]))
    roof["kernel"] = dom_name
    roof["peak_source"] = ("pinned cudaMemcpy H2D measured in this run" if roof["bound"] == "pcie"
                           else f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})")

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = reference_sample(args, steps=3, warmup=1, threads=cpu_threads(args))
        cpu_baseline = {kk: cb[kk] for kk in ("value", "unit", "cores", "kind", "sample", "extrapolation",
                                              "cpu_model")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if shard_heads else "weak", "vs_baseline": None,
            "dtype": kvd, "data": "synthetic",
            "config": workload_config(args, plan_info, world), "numa": numa,
            "hit_ratio": hits / max(1, hits + misses),
            "step_ms": {"min": min(step_ms), "p50": statistics.median(step_ms), "max": max(step_ms)},
            "pcie_gather_gbs_in_step": gathered / (ms / 1e3) / 1e9,
            "pcie_link_peak_gbs": best, "pcie_gen5_x16_theoretical_gbs": 64.0,
            "pcie_in_step_frac": {"of_memcpy_peak": gathered / (ms / 1e3) / 1e9 / best if best else None,
                                  "of_gen5_x16_theoretical": gathered / (ms / 1e3) / 1e9 / 64.0},
            "per_kernel_ms": {kk: round(v["ms"], 4) for kk, v in sorted(per_kernel.items())},
            "roofline": roof, "rooflines": rooflines, "layer_timing": layer_timing,
            "e2e": e2e, "gpu_launches": launches, "kernels_per_step": eng.kernels_per_step(),
            "clocks": clocks.summary(), "cpu_baseline": cpu_baseline,
            "setup_s": setup_s, "prefill_s": prefill_s,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: re-run this script
    under torch.distributed.run with N ranks on this node (one process per
    GPU, rendezvous on 127.0.0.1), the way the reference's runner fans
    independent engines out over a worker pool (runner.cpp:186-278). Rank 0
    prints the JSON line; the launcher's exit code is returned."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
