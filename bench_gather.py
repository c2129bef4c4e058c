#!/usr/bin/env python3
"""BASELINE.json configs[4]: zero-copy gather sweep, 256-16384 selected rows per
head (bf16 K+V rows of d=128 = 256 B each, indices uniform-random distinct
sorted over n=131072), versus the reference's gather-copy path
(TransferEngine::kGatherCopy, pipeline_sim.cpp:12-22: CPU threads gather rows
into a pinned staging buffer, then one cudaMemcpy H2D) and versus the link
peak (one contiguous pinned cudaMemcpy).

Each measurement moves the K and V rows of `heads` heads in one launch per
matrix (the engine batches every missed head of a layer the same way).
Engines: lsu = 16-byte zero-copy loads (the engine's kernel), tma = one
cp.async.bulk per row from pinned host memory.

  python bench_gather.py [--heads 32] [--reps 5] [--threads 16] [--gpus N]

Prints one JSON line per row count, then a summary line. With --gpus N, one
process per GPU runs the same sweep CONCURRENTLY (a barrier before every timed
repetition), each from its own pinned host store bound to its GPU's NUMA node,
so PCIe-switch uplink sharing shows up; each line then carries the per-GPU
rates and their aggregate.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


class _NoBarrier:
    def wait(self):
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1, help="concurrent per-GPU sweeps (one process per GPU)")
    ap.add_argument("--same-device", action="store_true", help="testing only: every worker on cuda:0")
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--threads", type=int, default=min(16, os.cpu_count() or 1))
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--rows", default="256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--huge", action="store_true", help="hugepage-backed pinned host store")
    ap.add_argument("--d", type=int, default=128, help="row width in bf16 elements (256 = K|V interleaved row)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--kv-one-launch", action="store_true",
                    help="K and V of the selected rows in ONE launch over one 2x store (the engine's access pattern)")
    ap.add_argument("--active", type=int, default=0,
                    help="gather from only this many (random) heads of the store (0 = all)")
    args = ap.parse_args()
    if args.gpus <= 1:
        results, peak = sweep(0, args, _NoBarrier(), emit=True)
        summarize([results], [peak], args)
        return
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(args.gpus)
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, args, barrier, q)) for r in range(args.gpus)]
    for p in procs:
        p.start()
    got = dict(q.get() for _ in procs)
    for p in procs:
        p.join()
        if p.exitcode:
            raise SystemExit(f"gather worker exited with {p.exitcode}")
    per = [got[r][0] for r in range(args.gpus)]
    peaks = [got[r][1] for r in range(args.gpus)]
    for i, line in enumerate(per[0]):
        rows = [p[i] for p in per]
        agg = {"rows_per_head": line["rows_per_head"], "gpus": args.gpus, "heads_per_gpu": line["heads"],
               "bytes_per_gpu": line["bytes"], "concurrent": True}
        for key in ("lsu", "tma", "cpu_staged"):
            if key + "_gbs" in line:
                agg[key + "_gbs_per_gpu"] = [round(x[key + "_gbs"], 3) for x in rows]
                # conservative: every GPU's bytes over the slowest GPU's time
                agg[key + "_gbs_aggregate"] = sum(x["bytes"] for x in rows) / (max(x[key + "_ms"] for x in rows) * 1e-3) / 1e9
        agg["link_peak_gbs_per_gpu"] = [round(p, 3) for p in peaks]
        print(json.dumps(agg), flush=True)
    summarize(per, peaks, args)


def _worker(rank, args, barrier, q):
    args.threads = max(1, args.threads // args.gpus)
    results, peak = sweep(rank, args, barrier, emit=False)
    q.put((rank, (results, peak)))


def summarize(per, peaks, args):
    flat = [x for r in per for x in r]
    print(json.dumps({"summary": f"zero-copy gather sweep (configs[4]), {args.gpus} GPU(s)"
                                 + (" concurrently" if args.gpus > 1 else ""),
                      "link_peak_gbs_pinned_memcpy": peaks if args.gpus > 1 else peaks[0],
                      "pcie_gen5_x16_theoretical_gbs": 64.0,
                      "best_lsu_gbs": max(x["lsu_gbs"] for x in flat),
                      "best_tma_gbs": max(x["tma_gbs"] for x in flat),
                      "best_lsu_gbs_aggregate": max(sum(r[i]["bytes"] for r in per) / max(r[i]["lsu_ms"] for r in per)
                                                    / 1e6 for i in range(len(per[0]))),
                      "best_tma_gbs_aggregate": max(sum(r[i]["bytes"] for r in per) / max(r[i]["tma_ms"] for r in per)
                                                    / 1e6 for i in range(len(per[0]))),
                      "best_cpu_staged_gbs": max((x.get("cpu_staged_gbs", 0.0) for x in flat))}),
          flush=True)


def sweep(rank, args, barrier, emit):
    import torch
    from paper_2511_14510_b200 import _lib
    from paper_2511_14510_b200.engine import device_numa_node
    lib = _lib.load()
    gpu = 0 if args.same_device else rank
    dev = torch.device("cuda", gpu)
    torch.cuda.set_device(dev)
    node = device_numa_node(gpu) if os.path.exists("/sys/devices/system/node/node1") else -1
    d, esz, n, H = args.d, 2, args.n, args.heads
    row_bytes = d * esz
    # host store: H heads x n rows, K and V, pinned + mapped
    nbytes = H * n * row_bytes
    ptrs = []
    for _ in range(2):
        p = C.c_void_p()
        _lib.check(lib.clo_host_alloc_numa(nbytes, _lib.HOST_HUGEPAGES if args.huge else 0, node, C.byref(p)))
        ptrs.append(p.value)
        arr = np.frombuffer((C.c_char * nbytes).from_address(p.value), dtype=np.uint16)
        arr[:] = np.random.default_rng(len(ptrs)).integers(0, 65535, arr.size, dtype=np.uint16)
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    err = torch.zeros(1, dtype=torch.int32, device=dev)

    # link peak: contiguous pinned memcpy of 1 GiB
    pin = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    peak = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier.wait()  # with --gpus N: every GPU's link under load at once
        a.record(stream)
        dbuf.copy_(pin, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        peak = max(peak, (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9)
    del pin, dbuf

    rng = np.random.default_rng(7)
    results = []
    for r in [int(x) for x in args.rows.split(",")]:
        heads = sorted(rng.choice(H, args.active, replace=False)) if args.active else range(H)
        idx = np.concatenate([np.sort(rng.choice(n, r, replace=False)) + h * n for h in heads]).astype(np.int32)
        didx = torch.from_numpy(idx).to(dev)
        nsel = len(idx)
        dst = torch.empty((2, nsel, d), dtype=torch.int16, device=dev)
        moved = 2 * nsel * row_bytes
        line = {"rows_per_head": r, "heads": H, "bytes": moved, "n": n, "hugepages": args.huge}
        if args.kv_one_launch:  # one store [2][H*n] rows: indices into K then V halves, one launch
            if not hasattr(sweep, "_kv"):
                p = C.c_void_p()
                _lib.check(lib.clo_host_alloc_numa(2 * nbytes, 0, node, C.byref(p)))
                sweep._kv = p.value
            didx2 = torch.cat([didx, didx + H * n])
            dst2 = torch.empty((2 * nsel, d), dtype=torch.int16, device=dev)
            best = None
            for rep in range(args.reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                barrier.wait()
                a.record(stream)
                _lib.check(lib.clo_gather_rows_ex(sweep._kv, _lib.DTYPE_BF16, d, 2 * H * n, didx2.data_ptr(), 2 * nsel,
                                                  dst2.data_ptr(), 0, args.ctas, err.data_ptr(), sp))
                b.record(stream)
                torch.cuda.synchronize()
                if rep:
                    best = a.elapsed_time(b) if best is None else min(best, a.elapsed_time(b))
            line["kv1_ms"] = best
            line["kv1_gbs"] = moved / (best * 1e-3) / 1e9
        for name, engine in (("lsu", 0), ("tma", 1)):
            best = None
            for rep in range(args.reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                barrier.wait()
                a.record(stream)
                for m in range(2):
                    _lib.check(lib.clo_gather_rows_ex(ptrs[m], _lib.DTYPE_BF16, d, H * n, didx.data_ptr(), nsel,
                                                      dst[m].data_ptr(), engine, args.ctas, err.data_ptr(), sp))
                b.record(stream)
                torch.cuda.synchronize()
                if rep:
                    ms = a.elapsed_time(b)
                    best = ms if best is None else min(best, ms)
            assert int(err.item()) == 0
            # bit-exact check against the host rows
            hk = np.frombuffer((C.c_char * nbytes).from_address(ptrs[0]), dtype=np.uint16).reshape(H * n, d)
            got = dst[0].cpu().numpy().view(np.uint16)
            sample = np.arange(0, nsel, max(1, nsel // 257))
            assert np.array_equal(got[sample], hk[idx[sample]]), name
            line[f"{name}_ms"] = best
            line[f"{name}_gbs"] = moved / (best * 1e-3) / 1e9
        # gather-copy baseline: CPU threads gather into pinned staging, then H2D
        if args.skip_cpu:
            line["link_peak_gbs"] = peak
            line["lsu_frac_of_peak"] = line["lsu_gbs"] / peak
            results.append(line)
            if emit:
                print(json.dumps(line), flush=True)
            continue
        stg = C.c_void_p()
        _lib.check(lib.clo_host_alloc(nsel * row_bytes, C.byref(stg)))
        hidx = np.ascontiguousarray(idx)
        best = None
        for rep in range(min(args.reps, 3) + 1):
            torch.cuda.synchronize()
            barrier.wait()
            t0 = time.perf_counter()
            for m in range(2):
                _lib.check(lib.clo_gather_rows_cpu_staged(ptrs[m], _lib.DTYPE_BF16, d, H * n, hidx.ctypes.data, nsel,
                                                          stg.value, dst[m].data_ptr(), args.threads, sp))
                torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if rep:
                best = el if best is None else min(best, el)
        lib.clo_host_free(stg.value)
        line["cpu_staged_ms"] = best * 1e3
        line["cpu_staged_gbs"] = moved / best / 1e9
        line["cpu_threads"] = args.threads
        line["link_peak_gbs"] = peak
        line["lsu_frac_of_peak"] = line["lsu_gbs"] / peak
        line["tma_frac_of_peak"] = line["tma_gbs"] / peak
        results.append(line)
        if emit:
            print(json.dumps(line), flush=True)
    for p in ptrs:
        lib.clo_host_free(p)
    return results, peak


if __name__ == "__main__":
    main()
