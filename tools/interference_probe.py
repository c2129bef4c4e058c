"""Does a zero-copy PCIe gather slow down HBM-bound kernels running beside it?

Times an HBM-bound elementwise kernel (torch mul, 2 x 1 GiB of traffic) on one
stream, alone and while a long train of gather launches (clo_gather_rows_ex,
LSU or TMA variant) runs on a second stream. Prints one JSON line per case.
Run on a GPU box: python tools/interference_probe.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14510_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    H, n, d = 32, 131072, 128
    row = d * 2
    nbytes = H * n * row
    p = C.c_void_p()
    _lib.check(lib.clo_host_alloc(nbytes, C.byref(p)))
    np.frombuffer((C.c_char * nbytes).from_address(p.value), dtype=np.uint8)[:] = 1
    rng = np.random.default_rng(3)
    idx = np.concatenate([np.sort(rng.choice(n, 2048, replace=False)) + h * n for h in range(H)]).astype(np.int32)
    didx = torch.from_numpy(idx).to(dev)
    dst = torch.empty((len(idx), d), dtype=torch.int16, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    x = torch.ones(1 << 28, dtype=torch.float32, device=dev)  # 1 GiB
    y = torch.empty_like(x)
    s_g = torch.cuda.Stream(dev, priority=-1)
    s_h = torch.cuda.Stream(dev)

    def hbm_ms(reps=20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s_h):
            a.record(s_h)
            for _ in range(reps):
                torch.mul(x, 2.0, out=y)
            b.record(s_h)
        return a, b, reps

    def gathers(engine, launches, ctas=0):
        sp = C.c_void_p(s_g.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s_g)
        for _ in range(launches):
            _lib.check(lib.clo_gather_rows_ex(p.value, _lib.DTYPE_BF16, d, H * n, didx.data_ptr(), len(idx),
                                              dst.data_ptr(), engine, ctas, err.data_ptr(), sp))
        b.record(s_g)
        return a, b

    for _ in range(2):  # warm-up
        hbm_ms(2)
        gathers(0, 1)
        gathers(1, 1)
    torch.cuda.synchronize()
    a, b, reps = hbm_ms()
    torch.cuda.synchronize()
    alone = a.elapsed_time(b) / reps
    print(json.dumps({"case": "hbm alone", "ms": alone, "gbs": 2 * x.numel() * 4 / (alone * 1e-3) / 1e9}))
    # the engine's grids: LSU 48 CTAs x 256 threads, TMA 148 one-warp CTAs
    for name, engine, ctas in (("lsu", 0, 48), ("tma", 1, 148), ("lsu-1184", 0, 0)):
        ga, gb = gathers(engine, 1, ctas)
        torch.cuda.synchronize()
        g_alone = ga.elapsed_time(gb)
        ga, gb = gathers(engine, 40, ctas)  # long gather train
        a, b, reps = hbm_ms()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        g_ms = ga.elapsed_time(gb) / 40
        print(json.dumps({"case": f"hbm beside {name} gather", "ms": ms,
                          "gbs": 2 * x.numel() * 4 / (ms * 1e-3) / 1e9, "slowdown": ms / alone,
                          "gather_ms_alone": g_alone, "gather_ms_beside": g_ms,
                          "gather_gbs_alone": dst.numel() * 2 / (g_alone * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
