#!/usr/bin/env python
"""Direct launches vs CUDA-graph replays of the headline kernels under the
bench's timing rules (cold-and-clean L2 before every launch, events on the
launching stream): how much of the per-launch event time is launch
processing."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    s = wl.stencil27()
    n = s["nrows"]
    e = wl.csr_to_ell(s["pos"], s["crd"], s["vals"], n)
    p, c, v, x = T(s["pos"]), T(s["crd"]), T(s["vals"]), T(s["x"])
    ec, ev = T(e["crd"]), T(e["vals"])
    y = torch.empty(n, dtype=torch.float64, device=dev)
    timer = bench.KernelTimer(torch, K, 2 * bench.l2_bytes(torch))
    fns = {"csr": lambda: K.spmv_csr(n, n, p, c, v, x, y),
           "ell": lambda: K.spmv_ell(n, n, 27, ec, ev, x, y)}
    stream = torch.cuda.Stream()
    graphs = {}
    for k, fn in fns.items():
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        graphs[k] = g
    gfns = {f"{k}_graph": (lambda g=g: g.replay()) for k, g in graphs.items()}
    res = timer.run({**fns, **gfns}, 300, 5)
    for k, ts in res.items():
        print(f"{k:10s} {np.mean(ts) * 1e3:7.2f} us (median {np.median(ts) * 1e3:7.2f})", flush=True)


if __name__ == "__main__":
    main()
