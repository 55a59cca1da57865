"""Phase timestamps of the resident COO kernel (SL_CR_TIMING alt build)."""
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1804_10112_b200 import _lib, kernels as K, workloads as wl  # noqa: E402

d = wl.coo_spmv()
n, m = d["nrows"], d["ncols"]
T = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
r, c, v, x = T(d["rows"]), T(d["cols"]), T(d["vals"]), T(d["x"])
y = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(5):
    K.spmv_coo(n, m, r, c, v, x, y)
torch.cuda.synchronize()
buf = np.zeros(160 * 12, dtype=np.uint64)
L = _lib.load()
L.sl_debug_coo_resident_times(buf.ctypes.data_as(ctypes.c_void_p))
t = buf.reshape(160, 12)[:148].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = ["start"] + [f"chunk{i}" for i in range(7)] + ["products", "slice0"]
for i, nm in enumerate(names):
    col = rel[:, i]
    print(f"{nm:9s} min {col.min():7.2f} median {np.median(col):7.2f} max {col.max():7.2f} us")
