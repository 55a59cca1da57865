"""D3 DIA SpMV under bench.py's protocol (A/B of library builds via SL_LIB_PATH)."""
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
g = wl.dia7()
n = g["nrows"]
offs = np.asarray(g["offsets"], dtype=np.int32)
b = bench.bytes_dia(n, n, offs)
ops = bench.dev_copies(torch, (g["vals"], g["x"], np.empty(n)), bench.copies_for(b, l2), dev)
y0 = K.spmv_dia(n, n, offs, ops[0][0], ops[0][1]).clone()
timer = bench.KernelTimer(torch, K, l2)
tt = timer.run({"dia": [lambda o=o: K.spmv_dia(n, n, offs, o[0], o[1], o[2]) for o in ops]}, 30, 3)
print(f"DIA D3 {tt['dia'] * 1e3:.2f} us frac {b / tt['dia'] / 1e6 / 6554.6:.4f} "
      f"checksum {float(y0.sum()):.17g}")
