#!/usr/bin/env python
"""SpMM on power-law rows: the group kernel alone vs the long-row split
(sl_spmm_csr_split_f64), event time per launch and bit-equality of the two.

    python tools/spmm_skew_prof.py [--rows 200000] [--K 16]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1804_10112_b200 import kernels as K  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=200_000)
    ap.add_argument("--K", type=int, nargs="+", default=[8, 16, 32])
    args = ap.parse_args()
    rng = np.random.default_rng(5)
    n = m = args.rows
    lens = np.minimum((rng.pareto(1.1, n) * 8).astype(np.int64), m // 2)
    pos = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=pos[1:])
    nnz = int(pos[-1])
    rows_of = np.repeat(np.arange(n), lens)
    crd = rng.integers(0, m, nnz).astype(np.int64)
    order = np.lexsort((crd, rows_of))
    crd = crd[order].astype(np.int32)        # duplicates allowed: sorted within rows
    vals = rng.uniform(-1, 1, nnz)
    print(f"rows {n}, nnz {nnz}, longest row {lens.max()}, rows > 1024: {(lens > 1024).sum()}")
    d = torch.device("cuda", 0)
    P = torch.as_tensor(pos.astype(np.int32), device=d)
    C = torch.as_tensor(crd, device=d)
    V = torch.as_tensor(vals, device=d)
    for Kc in args.K:
        X = torch.as_tensor(rng.uniform(-1, 1, (m, Kc)), device=d)
        Y0 = K.spmm_csr(n, m, P, C, V, X)
        Y1 = K.spmm_csr(n, m, P, C, V, X, long_min=1024)
        same = bool(torch.equal(Y0.view(-1).view(torch.int64), Y1.view(-1).view(torch.int64)))
        t0 = timed(lambda: K.spmm_csr(n, m, P, C, V, X))
        line = f"K={Kc}: group kernel {t0:.1f} us"
        for lm in (256, 1024, 4096):
            t1 = timed(lambda: K.spmm_csr(n, m, P, C, V, X, long_min=lm))
            line += f"; split(long_min={lm}) {t1:.1f} us"
        print(line + f"; bit-equal {same}")


if __name__ == "__main__":
    main()
