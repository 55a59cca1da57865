"""A+B (D4) timing under bench.py's protocol (rotating copies, graph replay),
plus the per-launch ncu-friendly single call.  python tools/time_add.py [K]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = torch.device("cuda", 0)
a = wl.add_ab()
n = a["nrows"]
l2 = bench.l2_bytes(torch)
ops = bench.dev_copies(torch, (a["a_pos"], a["a_crd"], a["a_vals"], a["b_rows"], a["b_cols"],
                               a["b_vals"]), 5, dev)
outs = {}


def add(o, two_pass=False):
    outs["c"] = K.add_csr(n, o[0], o[1], o[2], o[4], o[5], b_rows=o[3], sync=False,
                          two_pass=two_pass)


timer = bench.KernelTimer(torch, K, l2)
tt = timer.run({"add": [lambda o=o: add(o) for o in ops]}, steps, 3)
nnz_c = int(outs["c"][0][n].item())
b = 4 * (n + 1) + 12 * len(a["a_crd"]) + 16 * len(a["b_cols"]) + 4 * (n + 1) + 12 * nnz_c
t = tt["add"]
print(f"A+B D4: {t * 1e3:.2f} us/launch  {b / t / 1e6:.1f} GB/s  frac {b / t / 1e6 / 6554.6:.4f}  "
      f"({timer.method})")
