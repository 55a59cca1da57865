#!/usr/bin/env python
"""A/B the COO SpMV kernels (SL_COO_SWP: 0 = K1 tiles, >0 = persistent K1b
with register prefetch at 4/6/8/5 blocks per SM) on D1 and on the 64^3
stencil as COO: bit-exactness against the default, then mean CUDA-event time
per launch with the bench's cold-and-clean L2 flush."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--cfgs", default="0,1,2,3,4")
    args = ap.parse_args()
    import bench
    timer = bench.KernelTimer(torch, K, 2 * bench.l2_bytes(torch))
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    d = wl.coo_spmv()
    s = wl.stencil27()
    srows = np.repeat(np.arange(s["nrows"], dtype=np.int32), np.diff(s["pos"]))
    rng = np.random.default_rng(3)
    ev_rows = np.sort(rng.integers(0, 50_000, 300_001)).astype(np.int32)   # odd nnz, empty rows
    ev_cols = rng.integers(0, 7_000, len(ev_rows)).astype(np.int32)
    mats = {"d1": (d["nrows"], d["ncols"], d["rows"], d["cols"], d["vals"], d["x"]),
            "stencil": (s["nrows"], s["nrows"], srows, s["crd"], s["vals"], s["x"]),
            "ragged": (50_000, 7_000, ev_rows, ev_cols, rng.uniform(-1, 1, len(ev_rows)),
                       rng.uniform(-1, 1, 7_000))}
    for name, (n, m, r, c, v, x) in mats.items():
        tr, tc, tv, tx = T(r), T(c), T(v), T(x)
        os.environ["SL_COO_SWP"] = "0"
        y0 = K.spmv_coo(n, m, tr, tc, tv, tx).clone()
        fns = {}
        for cfg in args.cfgs.split(","):
            os.environ["SL_COO_SWP"] = cfg
            y = torch.full((n,), float("nan"), dtype=torch.float64, device=dev)
            K.spmv_coo(n, m, tr, tc, tv, tx, y)
            torch.cuda.synchronize()
            print(f"{name} cfg {cfg}: bit-exact {torch.equal(y.view(torch.int64), y0.view(torch.int64))}")

            def f(cfg=cfg):
                os.environ["SL_COO_SWP"] = cfg
                K.spmv_coo(n, m, tr, tc, tv, tx)
            fns[cfg] = f
        if name == "ragged":
            continue
        res = timer.run(fns, args.reps, 5)
        b = 16 * len(r) + 8 * m + 8 * n
        for k, ts in res.items():
            ms = float(np.mean(ts))
            print(f"{name} cfg {k}: {ms * 1e3:8.2f} us  {b / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
