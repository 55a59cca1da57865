import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
import oracle as orc
from paper_1804_10112_b200 import kernels as K
rng = np.random.default_rng(2)
n, m = 20_000, 40_000
def rows_of(lens):
    cols = [np.sort(rng.choice(m, int(k), replace=False)) for k in lens]
    pos = np.zeros(n + 1, np.int64); pos[1:] = np.cumsum(lens)
    return pos.astype(np.int32), np.concatenate(cols).astype(np.int32)
la = np.minimum(rng.zipf(1.7, n) - 1, 3000); lb = np.minimum(rng.zipf(1.7, n) - 1, 3000)
a_pos, a_crd = rows_of(la); b_pos, b_cols = rows_of(lb)
b_rows = np.repeat(np.arange(n, dtype=np.int32), lb)
a_vals = rng.uniform(-1, 1, len(a_crd)); b_vals = rng.uniform(-1, 1, len(b_cols))
rp, rc, rv = orc.add_csr(n, a_pos, a_crd, a_vals, b_cols, b_vals, b_rows=b_rows)
T = lambda a: torch.as_tensor(a, device='cuda')
pos, crd, vals = K.add_csr(n, T(a_pos), T(a_crd), T(a_vals), T(b_cols), T(b_vals), b_rows=T(b_rows))
crd = crd.cpu().numpy(); bad = np.nonzero(crd != rc)[0]
print('pos equal', np.array_equal(pos.cpu().numpy(), rp), 'bad crd', len(bad))
rows = np.searchsorted(rp, bad, side='right') - 1
ur = np.unique(rows)
for r in ur[:8]:
    t = r // 128
    print('row', r, 'tile', t, 'lenA', la[r], 'lenB', lb[r], 'oversized', la[r] > 768 or lb[r] > 768,
          'tile A', a_pos[min((t+1)*128, n)] - a_pos[t*128], 'tile B', b_pos[min((t+1)*128, n)] - b_pos[t*128],
          'nbad', (rows == r).sum())
