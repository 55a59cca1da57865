"""A/B of the SpMM gather batch (edit spmm.cu's G = 16 case to switch on SL_SPMM_B)."""
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import numpy as np, torch
from paper_1804_10112_b200 import kernels as K, workloads as wl
import bench
timer = bench.KernelTimer(torch, K, 2 * bench.l2_bytes(torch))
dev = torch.device('cuda', 0)
s = wl.stencil27(); n = s['nrows']
T = lambda a: torch.as_tensor(a, device=dev)
p, c, v = T(s['pos']), T(s['crd']), T(s['vals'])
X = torch.rand((n, 16), dtype=torch.float64, device=dev)
os.environ['SL_SPMM_B'] = '4'; Y0 = K.spmm_csr(n, n, p, c, v, X).clone()
fns = {}
for b in ('2', '4', '8', '16'):
    os.environ['SL_SPMM_B'] = b
    Y = K.spmm_csr(n, n, p, c, v, X); torch.cuda.synchronize()
    print(b, 'bit-exact', torch.equal(Y.view(torch.int64), Y0.view(torch.int64)))
    def f(b=b):
        os.environ['SL_SPMM_B'] = b
        K.spmm_csr(n, n, p, c, v, X)
    fns[b] = f
res = timer.run(fns, 50, 3)
for k, ts in res.items(): print('spmm K=16 batch', k, round(float(np.mean(ts)) * 1e3, 2), 'us')
