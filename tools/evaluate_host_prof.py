#!/usr/bin/env python
"""Host-side cost of one `evaluate('y(i) = A(i,j) * x(j)')` call (the e2e
leg's per-step Python work): cProfile over many calls with a host x, sorted
by own time.

    python tools/evaluate_host_prof.py [--calls 3000]
"""

import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
from paper_1804_10112_b200.engine import evaluate  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=3000)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    st = wl.stencil27()
    n = st["nrows"]
    pos, crd, vals = (torch.as_tensor(a, device=dev) for a in (st["pos"], st["crd"], st["vals"]))
    A = F.csr_storage(pos, crd, vals, (n, n), device=dev)
    x = F.dense_storage(torch.as_tensor(st["x"]).pin_memory(), device=None)
    inputs = {"A": A, "x": x}
    expr = "y(i) = A(i,j) * x(j)"
    for _ in range(20):
        evaluate(expr, inputs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.calls):
        evaluate(expr, inputs)
    t = (time.perf_counter() - t0) / args.calls * 1e6
    torch.cuda.synchronize()
    print(f"evaluate() host us/call (host x, no sync): {t:.1f}")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(args.calls):
        evaluate(expr, inputs)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
