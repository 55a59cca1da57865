"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE.json names no public dataset: every config is synthetic, and these
generators reproduce its shapes and value distributions.
They return plain numpy arrays already laid out the way the reference's
``formats.assemble`` lays them out (formats.py:361-501), so the same arrays
feed the GPU path, the C oracle and (at small sizes) the reference itself.

Layouts (reference file:line):
  COO-SoA  rows = L0 crd, cols = L1 crd, row-major sorted   formats.py:132-133
  CSR      pos[N+1], crd[nnz] sorted per row               formats.py:126-127
  ELL      slot-major crd/vals [S*N], pad (col 0, 0.0)      formats.py:164-169, 322-335, 443-455
  DIA      sorted offsets, vals [D*N] at d*N+i              formats.py:170-175, 394, 405-412
  COO-3    i = L0 crd, j = L1 crd, k = L2 crd               formats.py:138-140
  CSF      3x (pos, crd)                                    formats.py:136-137
  hash     crd[W] (-1 empty), vals[W] by slot, ascending-
           coordinate insertion with linear probing         formats.py:413-441, levels.py:312-333
"""

from __future__ import annotations

import numpy as np

# One documented seed per config.
SEED_COO = 1001
SEED_STENCIL27 = 1002
SEED_DIA7 = 1003
SEED_ADD = 1004
SEED_MTTKRP = 1005
SEED_HASH = 1006

EMPTY = -1


def _unique(a):
    """Sorted unique values (sort-based; numpy's hash path is slow for int64)."""
    a = np.sort(a, kind="stable")
    if len(a) == 0:
        return a
    keep = np.empty(len(a), dtype=bool)
    keep[0] = True
    np.not_equal(a[1:], a[:-1], out=keep[1:])
    return a[keep]


def _fix_total(rng, lens, total, cap):
    """Adjust row lengths by +-1 at seeded random rows until sum == total."""
    lens = np.minimum(lens.astype(np.int64), cap)
    n = len(lens)
    for _ in range(10_000):
        diff = int(total - lens.sum())
        if diff == 0:
            return lens
        if diff > 0:
            cand = np.flatnonzero(lens < cap)
            pick = rng.choice(cand, size=min(diff, len(cand)), replace=False)
            lens[pick] += 1
        else:
            cand = np.flatnonzero(lens > 0)
            pick = rng.choice(cand, size=min(-diff, len(cand)), replace=False)
            lens[pick] -= 1
    raise ValueError(f"cannot reach {total} nonzeros with {n} rows capped at {cap}")


def _sample_rows_without_replacement(rng, lens, ncols, forbid=None):
    """Per row r, draw lens[r] distinct uniform columns (not in `forbid`).

    Returns row-major sorted int64 keys row*ncols + col.  `forbid` is a sorted
    key array whose entries may not be drawn.
    """
    n = len(lens)
    keys = np.empty(0, dtype=np.int64)
    need = lens.astype(np.int64).copy()
    for _ in range(200):
        tot = int(need.sum())
        if tot == 0:
            break
        rows = np.repeat(np.arange(n, dtype=np.int64), need)
        cand = rows * ncols + rng.integers(0, ncols, size=tot, dtype=np.int64)
        if forbid is not None and len(forbid):
            hit = np.searchsorted(forbid, cand)
            hit = np.minimum(hit, len(forbid) - 1)
            cand = cand[forbid[hit] != cand]
        keys = _unique(np.concatenate([keys, cand]))
        have = np.bincount(keys // ncols, minlength=n)
        # drop surplus (cannot happen) and recompute what is still missing
        need = lens - have
        if (need < 0).any():
            raise AssertionError("row overfilled")
    else:
        # dense-ish leftovers: exhaustive choice per row
        for r in np.flatnonzero(need > 0):
            taken = set((keys[keys // ncols == r] % ncols).tolist())
            if forbid is not None:
                taken |= set((forbid[forbid // ncols == r] % ncols).tolist())
            free = np.array(sorted(set(range(ncols)) - taken), dtype=np.int64)
            extra = rng.choice(free, size=int(need[r]), replace=False)
            keys = _unique(np.concatenate([keys, r * ncols + extra]))
    return keys


def coo_spmv(n=200_000, ncols=None, nnz=2_000_000, lam=10.0, seed=SEED_COO):
    """D1: Poisson(lam) row lengths adjusted to exactly nnz, uniform distinct
    columns per row, row-major sorted COO, vals and x ~ U[-1, 1]."""
    ncols = n if ncols is None else ncols
    rng = np.random.default_rng(seed)
    lens = _fix_total(rng, rng.poisson(lam, n), nnz, ncols)
    keys = _sample_rows_without_replacement(rng, lens, ncols)
    rows = (keys // ncols).astype(np.int32)
    cols = (keys % ncols).astype(np.int32)
    vals = rng.uniform(-1.0, 1.0, size=len(keys))
    x = rng.uniform(-1.0, 1.0, size=ncols)
    return dict(nrows=n, ncols=ncols, rows=rows, cols=cols, vals=vals, x=x)


def coo_to_csr_pos(rows, nrows):
    counts = np.bincount(rows, minlength=nrows)
    pos = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=pos[1:])
    return pos.astype(np.int32)


def stencil27(g=64, seed=SEED_STENCIL27, gz=None, z0=0, z1=None):
    """D2: 27-point stencil on a g x g x gz grid (gz = g by default),
    i = z*g^2 + y*g + x.  Diagonal 26, off-diagonals -1 + U[-0.01, 0.01];
    x ~ U[-1, 1].  Returns CSR arrays of the rows of z-planes [z0, z1)
    (the whole grid by default) with global column indices, and the global x.
    The z-slab form is the row block a rank owns in the multi-GPU run."""
    gz = g if gz is None else gz
    z1 = gz if z1 is None else z1
    rng = np.random.default_rng(seed)
    n = g * g * gz
    x = rng.uniform(-1.0, 1.0, size=n)
    rng = np.random.default_rng([seed, z0, z1])
    idx = np.arange(z0 * g * g, z1 * g * g, dtype=np.int64)
    z, y, xx = idx // (g * g), (idx // g) % g, idx % g
    cols, valid, isdiag = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((z + dz >= 0) & (z + dz < gz) & (y + dy >= 0) & (y + dy < g)
                      & (xx + dx >= 0) & (xx + dx < g))
                cols.append(idx + dz * g * g + dy * g + dx)
                valid.append(ok)
                isdiag.append(np.full(len(idx), dz == 0 and dy == 0 and dx == 0))
    cols = np.stack(cols, axis=1)          # (rows, 27), ascending per row
    valid = np.stack(valid, axis=1)
    isdiag = np.stack(isdiag, axis=1)
    crd = cols[valid].astype(np.int32)
    diag = isdiag[valid]
    vals = np.where(diag, 26.0, -1.0 + rng.uniform(-0.01, 0.01, size=len(crd)))
    pos = np.zeros(len(idx) + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=pos[1:])
    return dict(nrows=len(idx), ncols=n, row0=z0 * g * g, pos=pos.astype(np.int32), crd=crd,
                vals=vals, x=x)


def csr_to_ell(pos, crd, vals, nrows, nslots=0):
    """Slot-major ELL (formats.py:322-335, 443-455): slot s of row i holds the
    row's s-th stored entry at position s*N + i; padding is (col 0, 0.0)."""
    pos = pos.astype(np.int64)
    lens = np.diff(pos)
    s_max = int(lens.max(initial=0))
    S = max(s_max, nslots)
    ecrd = np.zeros((S, nrows), dtype=np.int32)
    evals = np.zeros((S, nrows), dtype=np.float64)
    rows = np.repeat(np.arange(nrows), lens)
    slot = np.arange(len(crd)) - np.repeat(pos[:-1], lens)
    ecrd[slot, rows] = crd
    evals[slot, rows] = vals
    return dict(nslots=S, crd=ecrd.reshape(-1), vals=evals.reshape(-1))


def dia7(g=128, seed=SEED_DIA7):
    """D3: 7-point Laplacian on a g^3 grid as DIA with sorted offsets
    {-g^2, -g, -1, 0, 1, g, g^2}; main 6.0, off-diagonals -1.0, 0.0 where the
    neighbour leaves the grid.  Out-of-range slots hold 0.0 (never read)."""
    rng = np.random.default_rng(seed)
    n = g ** 3
    offsets = np.array([-g * g, -g, -1, 0, 1, g, g * g], dtype=np.int32)
    idx = np.arange(n, dtype=np.int64)
    z, y, xx = idx // (g * g), (idx // g) % g, idx % g
    coord = {1: xx, g: y, g * g: z}
    vals = np.zeros((len(offsets), n), dtype=np.float64)
    for d, off in enumerate(offsets.tolist()):
        if off == 0:
            vals[d] = 6.0
            continue
        c = coord[abs(off)]
        step = 1 if off > 0 else -1
        inside = (c + step >= 0) & (c + step < g)
        vals[d] = np.where(inside, -1.0, 0.0)
    x = rng.uniform(-1.0, 1.0, size=n)
    return dict(nrows=n, ncols=n, offsets=offsets, vals=vals.reshape(-1), x=x)


def dia_from_coo(rows, cols, vals, nrows, ncols):
    """Generic DIA assembly: diagonal set = sorted distinct (c - r)."""
    offs = _unique(cols.astype(np.int64) - rows.astype(np.int64))
    dvals = np.zeros((len(offs), nrows), dtype=np.float64)
    d = np.searchsorted(offs, cols.astype(np.int64) - rows.astype(np.int64))
    np.add.at(dvals, (d, rows.astype(np.int64)), vals)
    return dict(offsets=offs.astype(np.int32), vals=dvals.reshape(-1))


def add_ab(n=1_000_000, ncols=None, nnz_a=5_000_000, nnz_b=5_000_000, lam=5.0,
           overlap=0.1, seed=SEED_ADD):
    """D4: A CSR and B COO, Poisson(lam) rows adjusted to exact totals.  Each
    B entry coincides with an unused column of A's row with probability
    `overlap` (if any is left), otherwise takes a fresh column outside both
    rows.  No duplicates.  Values ~ U[-1, 1]."""
    ncols = n if ncols is None else ncols
    rng = np.random.default_rng(seed)
    lens_a = _fix_total(rng, rng.poisson(lam, n), nnz_a, ncols)
    keys_a = _sample_rows_without_replacement(rng, lens_a, ncols)
    lens_b = _fix_total(rng, rng.poisson(lam, n), nnz_b, ncols)
    pos_a = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens_a, out=pos_a[1:])
    # overlapping part: random distinct entries of A's row
    flags = rng.random(int(lens_b.sum())) < overlap
    brow = np.repeat(np.arange(n, dtype=np.int64), lens_b)
    orow = brow[flags]
    has = lens_a[orow] > 0
    orow = orow[has]
    pick = pos_a[orow] + (rng.random(len(orow)) * lens_a[orow]).astype(np.int64)
    okeys = _unique(keys_a[pick])
    n_over = np.bincount(okeys // ncols, minlength=n)
    n_over = np.minimum(n_over, lens_b)
    # trim rows where more overlaps were drawn than B entries (cannot exceed by construction)
    fresh_lens = lens_b - n_over
    fkeys = _sample_rows_without_replacement(rng, fresh_lens, ncols, forbid=keys_a)
    keys_b = _unique(np.concatenate([okeys, fkeys]))
    assert len(keys_b) == int(lens_b.sum())
    vals_a = rng.uniform(-1.0, 1.0, size=len(keys_a))
    vals_b = rng.uniform(-1.0, 1.0, size=len(keys_b))
    return dict(nrows=n, ncols=ncols,
                a_pos=pos_a.astype(np.int32), a_crd=(keys_a % ncols).astype(np.int32),
                a_vals=vals_a,
                b_rows=(keys_b // ncols).astype(np.int32),
                b_cols=(keys_b % ncols).astype(np.int32), b_vals=vals_b,
                overlap=int(len(np.intersect1d(keys_a, keys_b, assume_unique=True))))


def _zipf_draw(rng, dim, s, size):
    p = (np.arange(dim, dtype=np.float64) + 1.0) ** (-s)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    u = rng.random(size)
    return np.minimum(np.searchsorted(cdf, u, side="right"), dim - 1).astype(np.int64)


def mttkrp(I=20_000, J=15_000, K=10_000, nnz=40_000_000, R=32, s=1.2,
           seed=SEED_MTTKRP):
    """D5: i, j ~ finite Zipf(s) on [0, dim), k uniform; deduplicated, then a
    uniform subsample of exactly nnz unique coordinates sorted
    lexicographically.  vals = 1 - U[0, 1) in (0, 1]; B, C ~ U[-1, 1]."""
    rng = np.random.default_rng(seed)
    keys = np.empty(0, dtype=np.int64)
    draw = int(nnz * 1.8) + 1024
    for _ in range(20):
        i = _zipf_draw(rng, I, s, draw)
        j = _zipf_draw(rng, J, s, draw)
        k = rng.integers(0, K, size=draw, dtype=np.int64)
        keys = _unique(np.concatenate([keys, (i * J + j) * K + k]))
        if len(keys) >= nnz:
            break
        draw = int((nnz - len(keys)) * 3) + 1024
    else:
        raise ValueError("could not draw enough unique coordinates")
    if len(keys) > nnz:
        keep = np.sort(rng.choice(len(keys), size=nnz, replace=False))
        keys = keys[keep]
    k = (keys % K).astype(np.int32)
    ij = keys // K
    j = (ij % J).astype(np.int32)
    i = (ij // J).astype(np.int32)
    vals = 1.0 - rng.random(nnz)
    B = rng.uniform(-1.0, 1.0, size=(J, R))
    C = rng.uniform(-1.0, 1.0, size=(K, R))
    return dict(I=I, J=J, K=K, R=R, i=i, j=j, k=k, vals=vals, B=B, C=C)


def coo3_to_csf(i, j, k, dims):
    """CSF = (compressed, compressed, compressed) over lexicographically
    sorted unique coordinates (formats.py:136-137, 456-496)."""
    i = i.astype(np.int64)
    j = j.astype(np.int64)
    nnz = len(i)
    if nnz == 0:
        z = np.zeros(1, dtype=np.int32)
        e = np.zeros(0, dtype=np.int32)
        return dict(pos0=np.array([0, 0], dtype=np.int32), crd0=e, pos1=z, crd1=e,
                    pos2=z, crd2=e)
    new_slice = np.ones(nnz, dtype=bool)
    new_slice[1:] = i[1:] != i[:-1]
    new_fiber = new_slice.copy()
    new_fiber[1:] |= j[1:] != j[:-1]
    fstart = np.flatnonzero(new_fiber)
    sstart = np.flatnonzero(new_slice)
    crd0 = i[sstart].astype(np.int32)
    crd1 = j[fstart].astype(np.int32)
    pos2 = np.append(fstart, nnz).astype(np.int32)
    fiber_slice = np.cumsum(new_slice)[fstart] - 1
    pos1 = np.zeros(len(sstart) + 1, dtype=np.int64)
    np.cumsum(np.bincount(fiber_slice, minlength=len(sstart)), out=pos1[1:])
    return dict(pos0=np.array([0, len(sstart)], dtype=np.int32), crd0=crd0,
                pos1=pos1.astype(np.int32), crd1=crd1, pos2=pos2,
                crd2=k.astype(np.int32))


def hash_insert_sequential(coords, width, nseg=1, parent=None):
    """Sequential linear-probing insertion in the given order
    (levels.py:312-333): home slot coord % W inside the parent's segment,
    first empty slot wins, re-inserting a present coordinate is a no-op.
    Returns (crd table, slot of each coordinate)."""
    crd = np.full(nseg * width, EMPTY, dtype=np.int32)
    parent = np.zeros(len(coords), dtype=np.int64) if parent is None else parent
    slots = np.empty(len(coords), dtype=np.int64)
    for e, (c, pp) in enumerate(zip(coords.tolist(), parent.tolist())):
        base = pp * width
        for step in range(width):
            q = base + (c + step) % width
            v = crd[q]
            if v == c or v == EMPTY:
                crd[q] = c
                slots[e] = q
                break
        else:
            raise OverflowError(f"hashed segment of width {width} is full")
    return crd, slots


def hash_vector(n=200_000, m=100_000, width=131_072, seed=SEED_HASH):
    """H1: hash-vector x over n with m stored coordinates (uniform subset),
    pinned width, built by ascending-coordinate insertion."""
    rng = np.random.default_rng(seed)
    coords = np.sort(rng.choice(n, size=m, replace=False)).astype(np.int64)
    xv = rng.uniform(-1.0, 1.0, size=m)
    crd, slots = hash_insert_sequential(coords, width)
    vals = np.zeros(width, dtype=np.float64)
    vals[slots] = xv
    return dict(n=n, width=width, crd=crd, vals=vals, coords=coords.astype(np.int32),
                xvals=xv)
