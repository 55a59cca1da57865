"""SpMM (CSR x dense) on the 64^3 stencil and D1 under bench.py's protocol
(A/B via SL_SPMM_VEC2=0/1, one process each)."""
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
timer = bench.KernelTimer(torch, K, l2)
T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
st = wl.stencil27()
n, nnz = st["nrows"], len(st["crd"])
d = wl.coo_spmv()
n1, nnz1 = d["nrows"], len(d["rows"])
pos1 = wl.coo_to_csr_pos(d["rows"], n1)
rng = np.random.default_rng(5)
fns, nbytes = {}, {}
for Kc in (8, 16, 32):
    b = 12 * nnz + 4 * (n + 1) + 16 * n * Kc
    nc = bench.copies_for(b, l2)
    ops = bench.dev_copies(torch, (st["pos"], st["crd"], st["vals"], rng.uniform(-1, 1, (n, Kc)),
                                   np.empty((n, Kc))), nc, dev)
    fns[f"stencil K={Kc}"] = [lambda o=o: K.spmm_csr(n, n, o[0], o[1], o[2], o[3], Y=o[4]) for o in ops]
    nbytes[f"stencil K={Kc}"] = b
b = 12 * nnz1 + 4 * (n1 + 1) + 16 * n1 * 16
ops = bench.dev_copies(torch, (pos1, d["cols"], d["vals"], rng.uniform(-1, 1, (n1, 16)),
                               np.empty((n1, 16))), bench.copies_for(b, l2), dev)
fns["D1 K=16"] = [lambda o=o: K.spmm_csr(n1, n1, o[0], o[1], o[2], o[3], Y=o[4]) for o in ops]
nbytes["D1 K=16"] = b
tt = timer.run(fns, 20, 3)
for k, t in tt.items():
    print(f"{k:14s} {t * 1e3:8.2f} us  frac {nbytes[k] / t / 1e6 / 6554.6:.4f}")
