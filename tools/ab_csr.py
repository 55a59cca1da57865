#!/usr/bin/env python
"""A/B the CSR SpMV variants (and the ring-kernel configurations selected by
SL_CSR_RING) on the BASELINE stencil (D2a) and the D1 matrix: bit-exactness
against variant 0, then mean CUDA-event time per launch with the bench's
cold-and-clean L2 flush before every launch.

    python tools/ab_csr.py [--reps 200] [--cfgs 0,1,2,...]
"""

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
    ap.add_argument("--cfgs", default="0,1,2,3,4,5,6,7")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--var", type=int, default=4)
    ap.add_argument("--env", default="SL_CSR_RING")
    ap.add_argument("--mats", default="stencil27,d1,ragged")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    import bench
    timer = bench.KernelTimer(torch, K, 2 * bench.l2_bytes(torch))

    mats = {}
    s = wl.stencil27()
    mats["stencil27"] = (s["nrows"], s["pos"], s["crd"], s["vals"], s["x"])
    d = wl.coo_spmv()
    mats["d1"] = (d["nrows"], wl.coo_to_csr_pos(d["rows"], d["nrows"]), d["cols"], d["vals"], d["x"])
    # ragged edge case: long rows (> chunk), empty rows, odd alignment
    rng = np.random.default_rng(5)
    n = 5000
    lens = rng.integers(0, 40, n)
    lens[::97] = 0
    lens[5] = 5000
    lens[1234] = 3000
    pos = np.zeros(n + 1, np.int32)
    pos[1:] = np.cumsum(lens)
    crd = np.concatenate([np.sort(rng.choice(n, min(l, n), replace=False)) for l in lens]).astype(np.int32)
    pos[1:] = np.cumsum([min(l, n) for l in lens])
    mats["ragged"] = (n, pos, crd, rng.uniform(-1, 1, len(crd)), rng.uniform(-1, 1, n))

    for name, (n, pos, crd, vals, x) in mats.items():
        if name not in args.mats.split(","):
            continue
        p, c, v, xx = T(pos), T(crd), T(vals), T(x)
        y0 = K.spmv_csr(n, n, p, c, v, xx, variant=0).clone()
        nnz = len(crd)
        nbytes = 4 * (n + 1) + 12 * nnz + 16 * n
        fns = {"v0": lambda: K.spmv_csr(n, n, p, c, v, xx, variant=0),
               "v5": lambda: K.spmv_csr(n, n, p, c, v, xx, variant=5)}
        for cfg in args.cfgs.split(","):
            os.environ[args.env] = cfg
            y = K.spmv_csr(n, n, p, c, v, xx, variant=args.var)
            torch.cuda.synchronize()
            ok = torch.equal(y.view(torch.int64), y0.view(torch.int64))
            print(f"{name} ring cfg {cfg}: bit-exact vs v0: {ok}", flush=True)
            if not ok:
                bad = (y != y0).nonzero()[:5].flatten().tolist()
                print("   first mismatches", bad, y[bad].tolist(), y0[bad].tolist())

            def f(cfg=cfg):
                os.environ[args.env] = cfg
                K.spmv_csr(n, n, p, c, v, xx, variant=args.var)
            fns[f"ring{cfg}"] = f
        if name == "ragged":
            continue
        res = timer.run(fns, args.reps, args.warmup)
        for k, ts in res.items():
            ms = float(np.mean(ts))
            print(f"{name:10s} {k:7s} {ms * 1e3:8.2f} us  {nbytes / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
