#!/usr/bin/env python
"""Measure the L2 -> SM ceilings that bound MTTKRP (gathers of 256-byte factor
rows from an L2-resident table) and L2-resident streaming, on this B200.

    python tools/calib_l2.py            # builds tools/_calib_l2.so with nvcc

Prints one JSON line; bench.py reads profiles/l2_calib.json if present."""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
SO = HERE / "_calib_l2.so"


def build():
    src = HERE / "calib_l2.cu"
    if not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                        "-Xcompiler", "-fPIC", str(src), "-o", str(SO)], check=True)
    return ctypes.CDLL(str(SO))


def main():
    L = build()
    dev = torch.device("cuda", 0)
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    res = {"sm_count": sm}

    def timeit(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)) * 1e-3

    # random 256-byte rows of a 10000 x 32 f64 table (MTTKRP D5's C), 40M gathers
    K, n = 10_000, 40_000_000
    table = torch.randn(K * 32, dtype=torch.float64, device=dev)
    idx = torch.randint(0, K, (n,), dtype=torch.int32, device=dev)
    for blocks in (sm * 4, sm * 8):
        t = timeit(lambda: L.calib_gather_rows(ctypes.c_void_p(table.data_ptr()),
                                               ctypes.c_void_p(idx.data_ptr()), ctypes.c_int64(n),
                                               ctypes.c_void_p(out.data_ptr()), blocks,
                                               ctypes.c_void_p(s)))
        gbs = n * 256 / t / 1e9
        res[f"gather256_rows_{blocks}blk_GBs"] = round(gbs, 1)
    res["gather256_GBs"] = max(v for k, v in res.items() if k.startswith("gather256_rows"))
    # random 8-byte gathers from a 1.6 MB x (SpMV D1's x), 2M gathers, x warm in L2
    x = torch.randn(200_000, dtype=torch.float64, device=dev)
    ix = torch.randint(0, x.numel(), (2_000_000,), dtype=torch.int32, device=dev)
    best = 0.0
    for blocks in (sm * 2, sm * 4, sm * 8):
        t = timeit(lambda: L.calib_gather8(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(ix.data_ptr()),
                                           ctypes.c_int64(ix.numel()), ctypes.c_void_p(out.data_ptr()),
                                           blocks, ctypes.c_void_p(s)))
        best = max(best, ix.numel() / t / 1e9)
        res[f"gather8_2M_{blocks}blk_us"] = round(t * 1e6, 2)
    res["gather8_G_per_s"] = round(best, 1)
    # the same at 10x the count: separates throughput from the fixed
    # launch/ramp/event cost of a ~20 us kernel
    ix20 = torch.randint(0, x.numel(), (20_000_000,), dtype=torch.int32, device=dev)
    best20 = 0.0
    for blocks in (sm * 4, sm * 8, sm * 16):
        t = timeit(lambda: L.calib_gather8(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(ix20.data_ptr()),
                                           ctypes.c_int64(ix20.numel()), ctypes.c_void_p(out.data_ptr()),
                                           blocks, ctypes.c_void_p(s)))
        best20 = max(best20, ix20.numel() / t / 1e9)
        res[f"gather8_20M_{blocks}blk_us"] = round(t * 1e6, 2)
    res["gather8_20M_G_per_s"] = round(best20, 1)
    res["empty_kernel_event_us"] = round(timeit(lambda: L.calib_empty(sm, ctypes.c_void_p(s))) * 1e6, 2)
    # L2-resident stream (.cg), 32 MB buffer read 20 times
    buf = torch.randn(4 << 20, dtype=torch.float64, device=dev)
    reps = 20
    t = timeit(lambda: L.calib_stream_cg(ctypes.c_void_p(buf.data_ptr()), ctypes.c_int64(buf.numel()),
                                         reps, ctypes.c_void_p(out.data_ptr()), sm * 8,
                                         ctypes.c_void_p(s)))
    res["l2_stream_GBs"] = round(buf.numel() * 8 * reps / t / 1e9, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
