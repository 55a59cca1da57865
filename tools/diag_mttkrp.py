import sys, os, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import oracle
from paper_1804_10112_b200 import kernels as K, workloads as wl
m = wl.mttkrp(I=2000, J=1500, K=1000, nnz=400_000, R=32, seed=1)
ref, absA = oracle.mttkrp_coo3(2000, m['i'], m['j'], m['k'], m['vals'], m['B'], m['C'])
T = lambda a: torch.as_tensor(a, device='cuda')
A = K.mttkrp_coo3(2000, 1500, 1000, T(m['i']), T(m['j']), T(m['k']), T(m['vals']), T(m['B']), T(m['C'])).cpu().numpy()
err = np.abs(A - ref) / np.maximum(np.maximum(np.abs(ref), absA), 1e-300)
bad = np.argwhere(err > 1e-12)
rows = np.unique(bad[:, 0])
print(os.environ.get('SL_MTTKRP_NOREUSE'), 'bad entries', len(bad), 'bad rows', len(rows), rows[:10], 'max', err.max())
cnt = np.bincount(m['i'], minlength=2000)
print('nnz of bad rows', cnt[rows[:10]])
starts = np.concatenate([[0], np.cumsum(cnt)])
print('row starts', starts[rows[:10]], 'chunk of start', starts[rows[:10]] // 2048, 'end', (starts[rows[:10]+1]-1)//2048)
if len(bad): r, c = bad[0]; print('example', r, c, A[r, c], ref[r, c])
