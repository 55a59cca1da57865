#!/usr/bin/env python
"""A/B the ELL SpMV launch configurations (SL_ELL_CFG) on the 64^3 stencil:
bit-exactness against the default, then mean CUDA-event time per launch with
the bench's cold-and-clean L2 flush before every launch."""
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
    args = ap.parse_args()
    import bench
    timer = bench.KernelTimer(torch, K, 2 * bench.l2_bytes(torch))
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    s = wl.stencil27()
    n = s["nrows"]
    e = wl.csr_to_ell(s["pos"], s["crd"], s["vals"], n)
    ec, ev, x = T(e["crd"]), T(e["vals"]), T(s["x"])
    os.environ["SL_ELL_CFG"] = "0"
    y0 = K.spmv_ell(n, n, 27, ec, ev, x).clone()
    fns = {}
    for cfg in args.cfgs.split(","):
        os.environ["SL_ELL_CFG"] = cfg
        y = K.spmv_ell(n, n, 27, ec, ev, x)
        torch.cuda.synchronize()
        print(f"cfg {cfg}: bit-exact {torch.equal(y.view(torch.int64), y0.view(torch.int64))}")

        def f(cfg=cfg):
            os.environ["SL_ELL_CFG"] = cfg
            K.spmv_ell(n, n, 27, ec, ev, x)
        fns[cfg] = f
    res = timer.run(fns, args.reps, 5)
    b = 12 * 27 * n + 16 * n
    for k, ts in res.items():
        ms = float(np.mean(ts))
        print(f"ell cfg {k}: {ms * 1e3:8.2f} us  {b / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
