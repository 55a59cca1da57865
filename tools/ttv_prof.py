"""CSR SpMV variants on the D5 tensor's fibres (TTV's per-fibre reduction:
5.1M rows, Zipf-skewed lengths up to 9231)."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_10112_b200 import kernels as K, workloads as wl  # noqa: E402

t = wl.mttkrp()
csf = wl.coo3_to_csf(t['i'], t['j'], t['k'], None)
T = lambda a: torch.as_tensor(a, device='cuda')  # noqa: E731
p2, c2 = T(csf['pos2']), T(csf['crd2'])
tv = T(t['vals'])
v = T(np.random.default_rng(3).uniform(-1, 1, t['K']))
nf = len(csf['crd1'])
y0 = K.spmv_csr(nf, t['K'], p2, c2, tv, v, variant=5).clone()
alt = bool(K.L().sl_build_features() & 1)
for var in ((0, 1, 2, 4, 5, 6) if alt else (0, 2, 5, 6)):
    y = K.spmv_csr(nf, t['K'], p2, c2, tv, v, variant=var)
    torch.cuda.synchronize()
    ok = torch.equal(y.view(torch.int64), y0.view(torch.int64))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        K.spmv_csr(nf, t['K'], p2, c2, tv, v, y, variant=var)
    e1.record()
    torch.cuda.synchronize()
    print(f"variant {var}: {e0.elapsed_time(e1) / 3 * 1e3:9.1f} us  bit-exact vs K2a {ok}", flush=True)

# the same fibres as a row-sorted COO (rows = fibre index): the COO kernel's
# cross-tile row continuation on power-law rows
rows = T(np.repeat(np.arange(nf, dtype=np.int32), np.diff(csf['pos2'])))
yc = K.spmv_coo(nf, t['K'], rows, c2, tv, v)
torch.cuda.synchronize()
okc = torch.equal(yc.view(torch.int64), y0.view(torch.int64))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    K.spmv_coo(nf, t['K'], rows, c2, tv, v, yc)
e1.record()
torch.cuda.synchronize()
print(f"COO on the fibres: {e0.elapsed_time(e1) / 3 * 1e3:9.1f} us  bit-exact vs K2a {okc}", flush=True)
