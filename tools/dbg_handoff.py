import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1804_10112_b200 import kernels as K, workloads as wl
t = wl.mttkrp(); csf = wl.coo3_to_csf(t['i'], t['j'], t['k'], None)
T = lambda a: torch.as_tensor(a, device='cuda')
pos = csf['pos2']; p2, c2 = T(pos), T(csf['crd2']); tv = T(t['vals'])
v = T(np.random.default_rng(3).uniform(-1, 1, t['K'])); nf = len(csf['crd1'])
y5 = K.spmv_csr(nf, t['K'], p2, c2, tv, v, variant=5).cpu().numpy()
y6 = K.spmv_csr(nf, t['K'], p2, c2, tv, v, variant=6).cpu().numpy()
bad = np.nonzero(y5.view(np.int64) != y6.view(np.int64))[0]
L = np.diff(pos)
print('mismatches', len(bad), 'of', nf)
for r in bad[:10]:
    tile = r // 32; rows = np.arange(tile*32, min(tile*32+32, nf))
    print(r, 'len', L[r], 'tile', tile, 'tile nnz', L[rows].sum(), 'max', L[rows].max(), 'pos', pos[tile*32], 'y5', y5[r], 'y6', y6[r])
# how many tiles affected, by category
tiles = np.unique(bad // 32)
cat = {'reg': 0, 'staged_long': 0, 'chunked': 0}
for tl in tiles:
    rows = np.arange(tl*32, min(tl*32+32, nf)); tn = pos[rows[-1]+1] - (pos[rows[0]] & ~3)
    if L[rows].max() <= 28 and tn <= 896: cat['reg'] += 1
    elif tn <= 896: cat['staged_long'] += 1
    else: cat['chunked'] += 1
print(cat)
