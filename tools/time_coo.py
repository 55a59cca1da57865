"""COO SpMV (D1) timing under bench.py's protocol; SL_COO_KERNEL=tile for the
staged-tile kernel.  Also checks bit-equality with the oracle.
python tools/time_coo.py [K]"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402  (checker)
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = torch.device("cuda", 0)
l2 = bench.l2_bytes(torch)
cases = {"D1": wl.coo_spmv()}
if len(sys.argv) > 2:
    cases["pareto"] = wl.coo_spmv(n=200_000, nnz=2_000_000, lam=10.0, seed=3)
for name, d in cases.items():
    n, m, nnz = d["nrows"], d["ncols"], len(d["rows"])
    b = bench.bytes_coo(n, m, nnz)
    ref, _ = oracle.spmv_coo(n, d["rows"], d["cols"], d["vals"], d["x"])
    for kern in [os.environ.get("SL_COO_KERNEL", "rowptr")] if "SL_COO_KERNEL" in os.environ else ("rowptr", "tile"):
        os.environ["SL_COO_KERNEL"] = kern
        ops = bench.dev_copies(torch, (d["rows"], d["cols"], d["vals"], d["x"], np.empty(n)),
                               bench.copies_for(b, l2), dev)
        timer = bench.KernelTimer(torch, K, l2)
        t = timer.run({"coo": [lambda o=o: K.spmv_coo(n, m, *o) for o in ops]}, steps, 3)["coo"]
        y = ops[0][4].cpu().numpy()
        ok = np.array_equal(y.view(np.int64), ref.view(np.int64))
        print(f"{name} {kern:5s}: {t * 1e3:6.2f} us  {b / t / 1e6:7.1f} GB/s  frac {b / t / 1e6 / 6554.6:.4f}"
              f"  bit-exact {ok}")
