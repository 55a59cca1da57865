#!/usr/bin/env python
"""Achievable HBM bandwidth vs transfer size on this B200 (L2 flushed before
each timed launch): torch copy_ (read+write) and sum (read-only), fp64."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1804_10112_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for mb in (16, 35, 64, 87, 150, 262, 512, 1024, 2048):
    n = mb * (1 << 20) // 8
    a = torch.rand(n, dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    res = []
    for name, fn, bytes_ in (("copy", lambda: b.copy_(a), 2 * n * 8), ("sum", lambda: a.sum(), n * 8)):
        ts = []
        for it in range(15):
            K.l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        res.append(f"{name} {t*1e3:8.1f}us {bytes_/t/1e6:7.0f}GB/s")
    print(f"{mb:5d} MB  " + "   ".join(res), flush=True)
