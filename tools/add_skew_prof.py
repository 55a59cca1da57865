"""A + B on power-law rows (Zipf lengths, some rows of thousands of
nonzeros): the tiles beyond the 768-element stage take the global merge."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402

rng = np.random.default_rng(7)
n, m = 1_000_000, 1_000_000


def csr(lens):
    cols = [np.sort(rng.choice(m, int(k), replace=False)) for k in lens]
    pos = np.zeros(n + 1, np.int64)
    pos[1:] = np.cumsum(lens)
    return pos.astype(np.int32), np.concatenate(cols).astype(np.int32)


kind = sys.argv[1] if len(sys.argv) > 1 else "zipf"
if kind == "zipf":
    la = np.minimum(rng.zipf(1.7, n) - 1, 5000)
    lb = np.minimum(rng.zipf(1.7, n) - 1, 5000)
else:                     # uniform but denser than the 128-row tile stage holds
    la, lb = rng.poisson(float(kind), n), rng.poisson(float(kind), n)
ap, ac = csr(la)
bp, bc = csr(lb)
brows = np.repeat(np.arange(n, dtype=np.int32), lb)
T = lambda a: torch.as_tensor(a, device='cuda')  # noqa: E731
args = (n, T(ap), T(ac), T(rng.uniform(-1, 1, len(ac))), T(bc), T(rng.uniform(-1, 1, len(bc))))
for _ in range(2):
    K.add_csr(*args, b_rows=T(brows), sync=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
K.add_csr(*args, b_rows=T(brows), sync=False)
e1.record()
torch.cuda.synchronize()
print(f"A+B {kind} rows: nnz A {len(ac)} B {len(bc)}, max row {la.max()}/{lb.max()}: "
      f"{e0.elapsed_time(e1) * 1e3:.1f} us")
