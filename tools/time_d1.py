"""D1 COO and CSR SpMV under bench.py's protocol (A/B via env knobs)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda", 0)
l2 = bench.l2_bytes(torch)
d = wl.coo_spmv()
n, m, nnz = d["nrows"], d["ncols"], len(d["rows"])
pos = wl.coo_to_csr_pos(d["rows"], n)
b = bench.bytes_coo(n, m, nnz)
ops = bench.dev_copies(torch, (d["rows"], d["cols"], d["vals"], d["x"], np.empty(n)),
                       bench.copies_for(b, l2), dev)
cops = bench.dev_copies(torch, (pos, d["cols"], d["vals"], d["x"], np.empty(n)),
                        bench.copies_for(bench.bytes_csr(n, nnz), l2), dev)
timer = bench.KernelTimer(torch, K, l2)
tt = timer.run({"coo": [lambda o=o: K.spmv_coo(n, m, *o) for o in ops],
                "csr": [lambda o=o: K.spmv_csr(n, m, *o) for o in cops]}, 30, 3)
print(f"D1 COO {tt['coo'] * 1e3:.2f} us frac {b / tt['coo'] / 1e6 / 6554.6:.4f}; "
      f"CSR {tt['csr'] * 1e3:.2f} us frac {bench.bytes_csr(n, nnz) / tt['csr'] / 1e6 / 6554.6:.4f}")
