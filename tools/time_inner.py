"""INNERPROD of D5 with itself / with every other nonzero (CUDA events, mean of 5)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1804_10112_b200 import kernels as K, workloads as wl  # noqa: E402

mt = wl.mttkrp()
I, J, Kd = mt["I"], mt["J"], mt["K"]
T = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
x = (T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"]))
z = tuple(t.clone() for t in x)
zh = tuple(t[::2].contiguous() for t in x)
for name, zz in (("Z = X", z), ("Z = X[::2]", zh), ("X[::2] . X", None)):
    a, b = (x, zz) if zz is not None else (zh, x)
    for _ in range(2):
        out = K.inner_coo3(I, J, Kd, a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out = K.inner_coo3(I, J, Kd, a, b)
    e1.record()
    torch.cuda.synchronize()
    nb = 20 * (a[0].numel() + b[0].numel())
    t = e0.elapsed_time(e1) / 5
    print(f"{name:12s} {t:7.3f} ms  {nb / t / 1e6:7.1f} GB/s  value {float(out[0]):.17g}")
