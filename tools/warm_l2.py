#!/usr/bin/env python
"""Kernel time with the operands L2-resident: N back-to-back launches between
two events (no flush, no host gaps), per-launch mean.  Separates what a
kernel's own structure costs (latency chains, issue, shared memory) from the
HBM stream it has under the cold-L2 bench timing.

    python tools/warm_l2.py [--n 50]
"""

import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    jobs = {}
    s = wl.stencil27()
    n = s["nrows"]
    p, c, v, x = T(s["pos"]), T(s["crd"]), T(s["vals"]), T(s["x"])
    y = torch.empty(n, dtype=torch.float64, device=dev)
    e = wl.csr_to_ell(s["pos"], s["crd"], s["vals"], n)
    ec, ev = T(e["crd"]), T(e["vals"])
    bc = 4 * (n + 1) + 12 * len(s["crd"]) + 16 * n
    for var in (0, 4, 5):
        jobs[f"csr_v{var}"] = (bc, lambda var=var: K.spmv_csr(n, n, p, c, v, x, y, variant=var))
    jobs["ell"] = (12 * 27 * n + 16 * n, lambda: K.spmv_ell(n, n, 27, ec, ev, x, y))
    d = wl.coo_spmv()
    n1 = d["nrows"]
    r1, c1, v1, x1 = T(d["rows"]), T(d["cols"]), T(d["vals"]), T(d["x"])
    p1 = T(wl.coo_to_csr_pos(d["rows"], n1))
    y1 = torch.empty(n1, dtype=torch.float64, device=dev)
    jobs["coo_d1"] = (35_200_000, lambda: K.spmv_coo(n1, n1, r1, c1, v1, x1, y1))
    jobs["csr_d1"] = (4 * (n1 + 1) + 12 * len(d["rows"]) + 16 * n1,
                      lambda: K.spmv_csr(n1, n1, p1, c1, v1, x1, y1))
    for name, (b, fn) in jobs.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / args.n
        print(f"{name:8s} L2-warm back-to-back: {t * 1e3:7.2f} us/launch  ({b / t / 1e6:7.1f} GB/s)",
              flush=True)


if __name__ == "__main__":
    main()
