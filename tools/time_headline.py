"""Headline CSR / ELL kernels under bench.py's protocol (A/B via env knobs)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
dev = torch.device("cuda", 0)
l2 = bench.l2_bytes(torch)
st = wl.stencil27()
n, nnz = st["nrows"], len(st["crd"])
ell = wl.csr_to_ell(st["pos"], st["crd"], st["vals"], n)
bc, be = bench.bytes_csr(n, nnz), bench.bytes_ell(n, ell["nslots"])
y = torch.empty(n, dtype=torch.float64)
cops = bench.dev_copies(torch, (st["pos"], st["crd"], st["vals"], st["x"], y), bench.copies_for(bc, l2), dev)
eops = bench.dev_copies(torch, (ell["crd"], ell["vals"], st["x"], y), bench.copies_for(be, l2), dev)
timer = bench.KernelTimer(torch, K, l2)
tt = timer.run({"csr": [lambda o=o: K.spmv_csr(n, n, *o) for o in cops],
                "ell": [lambda o=o: K.spmv_ell(n, n, 27, *o) for o in eops]}, steps, 3)
print(f"CSR {tt['csr'] * 1e3:.2f} us ({bc / tt['csr'] / 1e6 / 6554.6:.4f})  "
      f"ELL {tt['ell'] * 1e3:.2f} us ({be / tt['ell'] / 1e6 / 6554.6:.4f})")
