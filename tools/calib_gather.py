#!/usr/bin/env python
"""Random-gather throughput on this B200: y = x[idx] (torch.index_select and
torch.take), idx = D1's column indices, L2 flushed before each launch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
d = wl.coo_spmv()
x = torch.as_tensor(d["x"], device=dev)
for name, idx in (("random(D1 cols)", torch.as_tensor(d["cols"].astype(np.int64), device=dev)),
                  ("sorted", torch.sort(torch.as_tensor(d["cols"].astype(np.int64), device=dev))[0]),
                  ("stencil-like", (torch.arange(2_000_000, device=dev) // 10) % x.numel())):
    ts = []
    for it in range(15):
        K.l2_flush(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.index_select(x, 0, idx)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    print(f"{name:18s} index_select 2M f64: {t*1e3:8.2f} us  ({2e6/t/1e6:.1f} G gathers/s)", flush=True)
