#!/usr/bin/env python
"""Where the end-to-end SpMV step's time goes (bench.py's `e2e` leg): host
cost of one evaluate() call, pinned H2D / D2H copy times of x and y, and the
full step loop over 2, 3, 4 and 6 streams.

    python tools/e2e_probe.py [--steps 200]
"""

import argparse
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
from paper_1804_10112_b200.engine import evaluate  # noqa: E402


def wall(fn, steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        fn(k)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    st = wl.stencil27()
    n = st["nrows"]
    pos, crd, vals = (torch.as_tensor(a, device=dev) for a in (st["pos"], st["crd"], st["vals"]))
    A = F.csr_storage(pos, crd, vals, (n, n), device=dev)
    xh = [torch.as_tensor(st["x"]).pin_memory() for _ in range(6)]
    yh = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(6)]
    xd = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    yd = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    xs_host = [F.dense_storage(x, device=None) for x in xh]
    xs_dev = [F.dense_storage(x, device=dev) for x in xd]
    streams = [torch.cuda.Stream(device=dev) for _ in range(6)]
    expr = "y(i) = A(i,j) * x(j)"
    for k in range(5):
        evaluate(expr, {"A": A, "x": xs_host[0]})
    torch.cuda.synchronize()

    # host cost of evaluate() with device-resident x (no copies), no sync
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        evaluate(expr, {"A": A, "x": xs_dev[0]})
    t_host = (time.perf_counter() - t0) / args.steps * 1e6
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        K.spmv_csr(n, n, pos, crd, vals, xd[0], yd[0])
    t_raw = (time.perf_counter() - t0) / args.steps * 1e6
    print(f"host us per evaluate() call (device x): {t_host:.1f}; per raw kernels.spmv_csr: {t_raw:.1f}")
    print(f"device-resident evaluate loop: {wall(lambda k: evaluate(expr, {'A': A, 'x': xs_dev[0]}), args.steps):.1f} us/step")
    print(f"H2D x only: {wall(lambda k: xd[0].copy_(xh[0], non_blocking=True), args.steps):.1f} us/step")
    print(f"D2H y only: {wall(lambda k: yh[0].copy_(yd[0], non_blocking=True), args.steps):.1f} us/step")

    def h2d_d2h(k):
        with torch.cuda.stream(streams[0]):
            xd[0].copy_(xh[0], non_blocking=True)
        with torch.cuda.stream(streams[1]):
            yh[1].copy_(yd[1], non_blocking=True)
    print(f"H2D + D2H on two streams: {wall(h2d_d2h, args.steps):.1f} us/step")

    for ns in (2, 3, 4, 6):
        def step(k, ns=ns):
            with torch.cuda.stream(streams[k % ns]):
                y = evaluate(expr, {"A": A, "x": xs_host[k % ns]}).vals
                yh[k % ns].copy_(y, non_blocking=True)
        print(f"e2e step (host x in, y out) over {ns} stream(s): {wall(step, args.steps):.1f} us/step")

        def step2(k, ns=ns):
            with torch.cuda.stream(streams[k % ns]):
                xd[k % ns].copy_(xh[k % ns], non_blocking=True)
                K.spmv_csr(n, n, pos, crd, vals, xd[k % ns], yd[k % ns])
                yh[k % ns].copy_(yd[k % ns], non_blocking=True)
        print(f"raw step (explicit copies + kernel) over {ns} stream(s): {wall(step2, args.steps):.1f} us/step")


if __name__ == "__main__":
    main()
