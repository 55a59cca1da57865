"""GPU parity: every kernel against the reference's golden vectors and the C
oracle on the same seeded inputs.

Bars: SpMV y and A+B (structure and values) bit-exact; MTTKRP within the
condition-scaled tolerance |gpu - ref| <= 1e-12 * max(|ref|, sum|terms|)
(north star: fp64 reductions within rtol 1e-12), plus run-to-run determinism.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

RTOL = 1e-12   # MTTKRP tolerance (condition-scaled)



# CSR SpMV variants in this build: the dispatch's (0 automatic, 2 merge-path,
# 5 row-block, 6 hand-off) and, in an SL_BUILD_ALT=1 build, the A/B ones
CSR_VARIANTS = [0, 2, 5, 6] + ([1, 3, 4] if K.L().sl_build_features() & 1 else [])

def cuda(a, dtype=None):
    a = np.asarray(a)
    if dtype is not None:
        a = a.astype(dtype)
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


# ---------------------------------------------------------------------------
# SpMV against the reference's goldens

def test_spmv_goldens_all_formats(golden):
    for name, c in golden["spmv"].items():
        nrows, ncols = int(c["nrows"]), int(c["ncols"])
        x = cuda(c["x"], np.float64)
        if "coo_y" in c:
            y = K.spmv_coo(nrows, ncols, cuda(c["coo_rows"], np.int32),
                           cuda(c["coo_cols"], np.int32), cuda(c["coo_vals"], np.float64), x)
            assert np.array_equal(bits(y), bits(c["coo_y"])), name
        if "csr_y" in c:
            for variant in CSR_VARIANTS:
                y = K.spmv_csr(nrows, ncols, cuda(c["csr_pos"], np.int32),
                               cuda(c["csr_crd"], np.int32), cuda(c["csr_vals"], np.float64), x,
                               variant=variant)
                assert np.array_equal(bits(y), bits(c["csr_y"])), (name, variant)
        if "ell_y" in c:
            y = K.spmv_ell(nrows, ncols, int(c["ell_nslots"]), cuda(c["ell_crd"], np.int32),
                           cuda(c["ell_vals"], np.float64), x)
            assert np.array_equal(bits(y), bits(c["ell_y"])), name
        if "dia_y" in c:
            y = K.spmv_dia(nrows, ncols, np.asarray(c["dia_offsets"], np.int32),
                           cuda(c["dia_vals"], np.float64), x)
            assert np.array_equal(bits(y), bits(c["dia_y"])), name
            y2 = K.spmv_dia(nrows, ncols, cuda(c["dia_offsets"], np.int32),
                            cuda(c["dia_vals"], np.float64), x)
            assert np.array_equal(bits(y2), bits(c["dia_y"])), name
        if "hash_y" in c:
            y = K.spmv_csr_hashx(nrows, cuda(c["csr_pos"], np.int32),
                                 cuda(c["csr_crd"], np.int32), cuda(c["csr_vals"], np.float64),
                                 int(c["hash_w"]), cuda(c["hash_crd"], np.int32),
                                 cuda(c["hash_vals"], np.float64))
            assert np.array_equal(bits(y), bits(c["hash_y"])), name
            y = K.spmv_csr_hashx(nrows, cuda(c["csr_pos"], np.int32),          # slot-map path
                                 cuda(c["csr_crd"], np.int32), cuda(c["csr_vals"], np.float64),
                                 int(c["hash_w"]), cuda(c["hash_crd"], np.int32),
                                 cuda(c["hash_vals"], np.float64), n=ncols)
            assert np.array_equal(bits(y), bits(c["hash_y"])), name


# ---------------------------------------------------------------------------
# SpMV against the oracle: medium, ragged and full BASELINE sizes

@pytest.mark.parametrize("n,nnz,lam,seed", [
    (3000, 30000, 10.0, 1), (5000, 200, 0.05, 2), (1, 4000, 1.0, 3), (20000, 20000, 1.0, 4),
    (777, 60000, 77.0, 5)])
def test_spmv_coo_csr_vs_oracle(orc, n, nnz, lam, seed):
    d = wl.coo_spmv(n=n, ncols=max(n, 4000), nnz=nnz, lam=lam, seed=seed)
    ref, _ = orc.spmv_coo(n, d["rows"], d["cols"], d["vals"], d["x"])
    x = cuda(d["x"])
    for direct in (False, True):       # row-pointer + hand-off path, staged-tile kernel
        y = K.spmv_coo(n, d["ncols"], cuda(d["rows"]), cuda(d["cols"]), cuda(d["vals"]), x,
                       direct=direct)
        assert np.array_equal(bits(y), bits(ref)), direct
    pos = wl.coo_to_csr_pos(d["rows"], n)
    for variant in CSR_VARIANTS:
        y = K.spmv_csr(n, d["ncols"], cuda(pos), cuda(d["cols"]), cuda(d["vals"]), x,
                       variant=variant)
        assert np.array_equal(bits(y), bits(ref)), variant
    e = wl.csr_to_ell(pos, d["cols"], d["vals"], n)
    y = K.spmv_ell(n, d["ncols"], e["nslots"], cuda(e["crd"]), cuda(e["vals"]), x)
    ref_e, _ = orc.spmv_ell(n, e["nslots"], e["crd"], e["vals"], d["x"])
    assert np.array_equal(bits(y), bits(ref_e))


def test_spmv_coo_long_rows_cross_tiles(orc):
    # rows far longer than one 2048-nonzero tile: the owner reads forward
    rows = np.repeat(np.arange(6, dtype=np.int32), [5000, 1, 0, 9000, 3, 0])
    rng = np.random.default_rng(0)
    cols = np.concatenate([np.sort(rng.choice(20000, k, replace=False)) for k in
                           [5000, 1, 0, 9000, 3, 0]]).astype(np.int32)
    vals = rng.uniform(-1, 1, len(rows))
    x = rng.uniform(-1, 1, 20000)
    ref, _ = orc.spmv_coo(8, rows, cols, vals, x)
    y = K.spmv_coo(8, 20000, cuda(rows), cuda(cols), cuda(vals), cuda(x))
    assert np.array_equal(bits(y), bits(ref))
    # the same rows through every CSR variant (row-stage: blocks far beyond
    # one staging round, rows cut by rounds)
    pos = wl.coo_to_csr_pos(rows, 8)
    for variant in CSR_VARIANTS:
        y = K.spmv_csr(8, 20000, cuda(pos), cuda(cols), cuda(vals), cuda(x), variant=variant)
        assert np.array_equal(bits(y), bits(ref)), variant


def test_spmv_csr_handoff_paths(orc):
    # 32-row tiles exercising each path of the register hand-off kernel: rows
    # <= 28 nonzeros (registers), a longer row inside the stage capacity (the
    # tile walks the stage), a tile beyond the capacity (warp per row), empty
    # rows and an empty tile, a partial last tile
    rng = np.random.default_rng(11)
    n, m = 230, 5000
    lens = rng.integers(0, 12, n)
    lens[3], lens[70], lens[100], lens[150] = 40, 29, 0, 200
    lens[160:192] = 30                      # 960 nonzeros in one tile: > 896
    lens[192:224] = 0                       # an empty tile
    cols = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for k in lens]).astype(np.int32)
    pos = np.zeros(n + 1, np.int32)
    pos[1:] = np.cumsum(lens)
    vals = rng.uniform(-1, 1, len(cols))
    x = rng.uniform(-1, 1, m)
    ref, _ = orc.spmv_csr(n, pos, cols, vals, x)
    for variant in [v for v in CSR_VARIANTS if v in (0, 4, 5, 6)]:
        y = cuda(np.full(n, np.nan))
        K.spmv_csr(n, m, cuda(pos), cuda(cols), cuda(vals), cuda(x), y=y, variant=variant)
        assert np.array_equal(bits(y), bits(ref)), variant


def test_spmv_csr_skewed_rows_many_tiles_per_block(orc):
    # power-law row lengths over enough rows that every persistent hand-off
    # block walks many tiles (grid = 12 blocks/SM): tiles of short rows, tiles
    # with a long row inside the stage, tiles far beyond it, empty tiles
    rng = np.random.default_rng(21)
    n, m = 200_000, 30_000
    lens = np.minimum(rng.zipf(1.6, n) - 1, 3000).astype(np.int64)
    lens[rng.random(n) < 0.01] = 0
    lens[150_000:150_064] = 0
    cols = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for k in lens]).astype(np.int32)
    pos = np.zeros(n + 1, np.int32)
    pos[1:] = np.cumsum(lens)
    vals = rng.uniform(-1, 1, len(cols))
    x = rng.uniform(-1, 1, m)
    ref, _ = orc.spmv_csr(n, pos, cols, vals, x)
    for variant in (0, 2, 5, 6):
        y = cuda(np.full(n, np.nan))
        K.spmv_csr(n, m, cuda(pos), cuda(cols), cuda(vals), cuda(x), y=y, variant=variant)
        assert np.array_equal(bits(y), bits(ref)), variant


def test_spmv_csr_misaligned_operands(orc):
    # crd/vals views starting one element in: the automatic choice falls back
    # to the row-block kernel; the row-stage kernel refuses (it bulk-copies
    # 16-byte granules)
    s = wl.stencil27(g=16)
    ref, _ = orc.spmv_csr(s["nrows"], s["pos"], s["crd"], s["vals"], s["x"])
    c = cuda(np.concatenate([[0], s["crd"]]).astype(np.int32))[1:]
    v = cuda(np.concatenate([[0.0], s["vals"]]))[1:]
    x = cuda(s["x"])
    y = K.spmv_csr(s["nrows"], s["ncols"], cuda(s["pos"]), c, v, x, variant=0)
    assert np.array_equal(bits(y), bits(ref))
    for variant in [v for v in CSR_VARIANTS if v in (4, 6)]:
        with pytest.raises(Exception):
            K.spmv_csr(s["nrows"], s["ncols"], cuda(s["pos"]), c, v, x, variant=variant)


def test_spmv_empty_matrix():
    x = cuda(np.ones(5))
    y = K.spmv_coo(9, 5, cuda(np.zeros(0, np.int32)), cuda(np.zeros(0, np.int32)),
                   cuda(np.zeros(0)), x)
    assert np.array_equal(bits(y), bits(np.zeros(9)))
    for variant in CSR_VARIANTS:     # y pre-filled with NaN: every row must be written
        y = cuda(np.full(9, np.nan))
        K.spmv_csr(9, 5, cuda(np.zeros(10, np.int32)), cuda(np.zeros(0, np.int32)),
                   cuda(np.zeros(0)), x, y=y, variant=variant)
        assert np.array_equal(bits(y), bits(np.zeros(9))), variant


def test_spmv_dia_vs_oracle_odd_shapes(orc):
    rng = np.random.default_rng(3)
    for nrows, ncols, offs in [(1000, 1300, [-999, -3, 0, 7, 1299]), (257, 100, [-256, -1, 0, 99]),
                               (5, 5, [-4, -2, 0, 2, 4]), (4096, 4096, list(range(-40, 41, 3)))]:
        offs = np.array(offs, dtype=np.int32)
        vals = rng.uniform(-1, 1, len(offs) * nrows)
        x = rng.uniform(-1, 1, ncols)
        ref, _ = orc.spmv_dia(nrows, ncols, offs, vals, x)
        y = K.spmv_dia(nrows, ncols, offs, cuda(vals), cuda(x))
        assert np.array_equal(bits(y), bits(ref)), (nrows, ncols)


@pytest.mark.slow
def test_full_size_spmv_bit_exact(orc):
    d = wl.coo_spmv()
    ref, _ = orc.spmv_coo(d["nrows"], d["rows"], d["cols"], d["vals"], d["x"])
    y = K.spmv_coo(d["nrows"], d["ncols"], cuda(d["rows"]), cuda(d["cols"]), cuda(d["vals"]),
                   cuda(d["x"]))
    assert np.array_equal(bits(y), bits(ref))
    s = wl.stencil27()
    ref, _ = orc.spmv_csr(s["nrows"], s["pos"], s["crd"], s["vals"], s["x"])
    x = cuda(s["x"])
    for variant in CSR_VARIANTS:
        y = K.spmv_csr(s["nrows"], s["ncols"], cuda(s["pos"]), cuda(s["crd"]), cuda(s["vals"]),
                       x, variant=variant)
        assert np.array_equal(bits(y), bits(ref)), variant
    e = wl.csr_to_ell(s["pos"], s["crd"], s["vals"], s["nrows"])
    ref_e, _ = orc.spmv_ell(s["nrows"], e["nslots"], e["crd"], e["vals"], s["x"])
    y = K.spmv_ell(s["nrows"], s["ncols"], e["nslots"], cuda(e["crd"]), cuda(e["vals"]), x)
    assert np.array_equal(bits(y), bits(ref_e))
    # ELL's padding terms 0.0*x[0] do not change finite results: ELL == CSR here
    assert np.array_equal(bits(ref_e), bits(ref))
    g = wl.dia7()
    ref, _ = orc.spmv_dia(g["nrows"], g["ncols"], g["offsets"], g["vals"], g["x"])
    y = K.spmv_dia(g["nrows"], g["ncols"], g["offsets"], cuda(g["vals"]), cuda(g["x"]))
    assert np.array_equal(bits(y), bits(ref))


# ---------------------------------------------------------------------------
# hashed level

@pytest.mark.parametrize("group", [1, 4, 8, 16, 32])
def test_hashed_locate_kats(level_kats, group):
    k = level_kats
    for tag, w in (("h4", 4), ("h8", 8), ("h16", 16)):
        pos, found = K.hashed_locate(cuda(k[f"{tag}_locate_q"], np.int32), w,
                                     cuda(k[f"{tag}_crd"], np.int32), group=group)
        assert np.array_equal(pos.cpu().numpy(), k[f"{tag}_locate_pos"]), (tag, group)
        assert np.array_equal(found.cpu().numpy().astype(np.int32), k[f"{tag}_locate_found"])
    pos, found = K.hashed_locate(cuda([7], np.int32), 4, cuda(k["hfull_crd"], np.int32),
                                 group=group)
    assert (int(pos[0]), int(found[0])) == tuple(k["hfull_locate_7"])
    w = int(k["hseg_w"])
    pos, found = K.hashed_locate(cuda(k["hseg_q_coord"], np.int32), w,
                                 cuda(k["hseg_crd"], np.int32),
                                 parent=cuda(k["hseg_q_parent"], np.int32), group=group)
    assert np.array_equal(pos.cpu().numpy(), k["hseg_q_pos"])
    assert np.array_equal(found.cpu().numpy().astype(np.int32), k["hseg_q_found"])


@pytest.mark.parametrize("group", [1, 8, 32])
def test_hashed_locate_vs_oracle_high_load(orc, group):
    h = wl.hash_vector(n=300_000, m=120_000, width=131_072, seed=9)   # load 0.92: long probes
    rng = np.random.default_rng(1)
    q = rng.integers(0, 300_000, 500_000).astype(np.int32)
    rp, rf = orc.hashed_locate(q, 131_072, h["crd"])
    pos, found = K.hashed_locate(cuda(q), 131_072, cuda(h["crd"]), group=group)
    assert np.array_equal(pos.cpu().numpy(), rp)
    assert np.array_equal(found.cpu().numpy().astype(bool), rf)


def test_hashed_insert_set_semantics(orc):
    rng = np.random.default_rng(5)
    w, nseg = 64, 50
    parent = rng.integers(0, nseg, 2000).astype(np.int32)
    coords = rng.integers(0, 200, 2000).astype(np.int32)
    crd, err = K.hashed_insert(cuda(coords), w, nseg=nseg, parent=cuda(parent), ordered=False)
    assert int(err.item()) == 0
    table = crd.cpu().numpy()
    ref, st = orc.hashed_insert(coords, w, nseg=nseg, parent=parent)
    assert st == 0
    for s in range(nseg):
        got = set(table[s * w:(s + 1) * w].tolist()) - {-1}
        exp = set(ref[s * w:(s + 1) * w].tolist()) - {-1}
        assert got == exp
    # every inserted coordinate is found through locate, nothing else is
    pos, found = K.hashed_locate(cuda(coords), w, crd, parent=cuda(parent))
    assert found.cpu().numpy().all()
    assert np.array_equal(table[pos.cpu().numpy()], coords)
    # overflow
    crd, err = K.hashed_insert(cuda(np.array([0, 2, 4], np.int32)), 2)
    assert int(err.item()) == 4


@pytest.mark.parametrize("w,nseg,n,crange,seed", [
    (64, 50, 2000, 200, 5),          # multi-segment, many repeats
    (4096, 1, 3000, 1 << 20, 6),     # one segment, scattered homes
    (1024, 1, 1000, 1024, 7),        # load ~0.63, heavy primary clustering
    (97, 3, 282, 10_000, 8),         # odd width, wrap-around probing, 94 per segment
    (131072, 1, 100_000, 200_000, 9)])  # H1's table (ascending-insert clusters)
def test_hashed_insert_ordered_exact_layout(orc, w, nseg, n, crange, seed):
    # the bulk insert builds exactly the table of sequential insert_coord calls
    rng = np.random.default_rng(seed)
    parent = rng.permutation(np.repeat(np.arange(nseg), -(-n // nseg))[:n]).astype(np.int32)
    coords = rng.integers(0, crange, n).astype(np.int32)
    if seed == 9:
        coords = np.sort(rng.choice(crange, n, replace=False)).astype(np.int32)
    half = n // 2
    # two calls: the second inserts into a table that already has entries
    crd, err = K.hashed_insert(cuda(coords[:half]), w, nseg=nseg, parent=cuda(parent[:half]))
    crd, err2 = K.hashed_insert(cuda(coords[half:]), w, nseg=nseg, parent=cuda(parent[half:]),
                                crd=crd)
    ref, st = orc.hashed_insert(coords, w, nseg=nseg, parent=parent)
    assert st == 0 and int(err.item()) == 0 and int(err2.item()) == 0
    assert np.array_equal(crd.cpu().numpy(), ref)


def test_hashed_insert_ordered_overflow():
    crd, err = K.hashed_insert(cuda(np.array([5, 7, 5, 9], np.int32)), 2)
    assert int(err.item()) == 4            # SL_ERR_HASH_SEGMENT_FULL: 3 distinct into width 2
    crd, err = K.hashed_insert(cuda(np.array([5, 7, 5, 7], np.int32)), 2)
    assert int(err.item()) == 0            # repeats are idempotent: exactly full
    assert sorted(crd.cpu().numpy().tolist()) == [5, 7]


def test_spmv_hashx_full_h1(orc):
    d = wl.coo_spmv()
    h = wl.hash_vector()
    pos = wl.coo_to_csr_pos(d["rows"], d["nrows"])
    ref, _ = orc.spmv_csr_hashx(d["nrows"], pos, d["cols"], d["vals"], h["width"], h["crd"],
                                h["vals"])
    y = K.spmv_csr_hashx(d["nrows"], cuda(pos), cuda(d["cols"]), cuda(d["vals"]), h["width"],
                         cuda(h["crd"]), cuda(h["vals"]))
    assert np.array_equal(bits(y), bits(ref))
    y = K.spmv_csr_hashx(d["nrows"], cuda(pos), cuda(d["cols"]), cuda(d["vals"]), h["width"],
                         cuda(h["crd"]), cuda(h["vals"]), n=d["ncols"])
    assert np.array_equal(bits(y), bits(ref))


def _map_vs_oracle(orc, crd, w, n, sample=None):
    m = K.hashed_slot_map(n, w, cuda(crd, np.int32)).cpu().numpy().view(np.uint64)
    q = np.arange(n, dtype=np.int32)
    if sample is not None:      # every stored coordinate plus a sample of the rest
        crd_a = np.asarray(crd)
        rng = np.random.default_rng(n)
        stored = crd_a[(crd_a >= 0) & (crd_a < n)]
        q = np.unique(np.concatenate([rng.choice(stored, min(sample, len(stored)), replace=False),
                                      rng.integers(0, n, sample)])).astype(np.int32)
        m = m[q]
    rp, rf = orc.hashed_locate(q, w, np.asarray(crd, np.int32))
    found = m != np.uint64(0xFFFFFFFFFFFFFFFF)
    assert np.array_equal(found, rf)
    assert np.array_equal((m[found] & np.uint64(0xFFFFFFFF)).astype(np.int64), rp[rf].astype(np.int64))


def test_hashed_slot_map_vs_probing(orc):
    """The slot map (one resolution per coordinate) equals per-query probing
    for tables built by insertion and for arbitrary contents: empty slots
    cutting probe paths, duplicates, a full table, wrap-around, one-slot tables."""
    h = wl.hash_vector()
    _map_vs_oracle(orc, h["crd"], h["width"], h["n"], sample=1500)
    h = wl.hash_vector(n=300_000, m=120_000, width=131_072, seed=9)
    _map_vs_oracle(orc, h["crd"], h["width"], h["n"], sample=1500)
    rng = np.random.default_rng(3)
    for w in (1, 2, 7, 1000, 5000):
        for fill in (0.0, 0.5, 0.9, 1.0):
            crd = np.where(rng.random(w) < fill, rng.integers(0, 3 * w + 1, w), -1).astype(np.int32)
            _map_vs_oracle(orc, crd, w, 3 * w + 2)
    crd = np.array([5, 5, -1, 5, 9, 1, 1, -1], np.int32)       # duplicates, gaps
    _map_vs_oracle(orc, crd, 8, 12)


# ---------------------------------------------------------------------------
# A + B

@pytest.mark.parametrize("two_pass", [False, True])
def test_add_goldens(golden, two_pass):
    for name, c in golden["add"].items():
        kw = {"b_pos": cuda(c["b_pos"], np.int32)} if "b_pos" in c else \
             {"b_rows": cuda(c["b_rows"], np.int32)}
        pos, crd, vals = K.add_csr(int(c["nrows"]), cuda(c["a_pos"], np.int32),
                                   cuda(c["a_crd"], np.int32), cuda(c["a_vals"], np.float64),
                                   cuda(c["b_cols"], np.int32), cuda(c["b_vals"], np.float64),
                                   two_pass=two_pass, **kw)
        assert np.array_equal(pos.cpu().numpy(), c["c_pos"]), name
        assert np.array_equal(crd.cpu().numpy(), c["c_crd"]), name
        assert np.array_equal(bits(vals), bits(c["c_vals"])), name


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("n,nnz,seed", [(2000, 9000, 1), (100_000, 500_000, 2), (70_000, 100, 3),
                                        (3000, 300_000, 4)])
def test_add_vs_oracle(orc, n, nnz, seed, two_pass):
    d = wl.add_ab(n=n, nnz_a=nnz, nnz_b=nnz, seed=seed)
    rp, rc, rv = orc.add_csr(n, d["a_pos"], d["a_crd"], d["a_vals"], d["b_cols"], d["b_vals"],
                             b_rows=d["b_rows"])
    pos, crd, vals = K.add_csr(n, cuda(d["a_pos"]), cuda(d["a_crd"]), cuda(d["a_vals"]),
                               cuda(d["b_cols"]), cuda(d["b_vals"]), b_rows=cuda(d["b_rows"]),
                               two_pass=two_pass)
    assert np.array_equal(pos.cpu().numpy(), rp)
    assert np.array_equal(crd.cpu().numpy(), rc)
    assert np.array_equal(bits(vals), bits(rv))


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("seed", [5, 6])
def test_add_duplicates_zeros_vs_oracle(orc, two_pass, seed):
    """B with repeated coordinates (grouped sums), explicit and signed zeros,
    rows of every length including ones past the stage capacity."""
    rng = np.random.default_rng(seed)
    n, m = 5000, 64
    la = rng.poisson(6, n)
    la[rng.integers(0, n, 3)] = 60                  # a few long rows
    a_pos = np.zeros(n + 1, np.int64)
    np.cumsum(np.minimum(la, m), out=a_pos[1:])
    a_crd = np.concatenate([np.sort(rng.choice(m, size=k, replace=False)) for k in np.diff(a_pos)])
    a_vals = rng.uniform(-1, 1, len(a_crd))
    a_vals[rng.random(len(a_vals)) < 0.05] = -0.0
    nb = 40000
    b_rows = np.sort(rng.integers(0, n, nb))
    b_rows[:3000] = 17                                # one row far past the capacity
    b_rows = np.sort(b_rows)
    b_cols = rng.integers(0, m, nb)
    o = np.lexsort((b_cols, b_rows))
    b_rows, b_cols = b_rows[o], b_cols[o]
    b_vals = rng.uniform(-1, 1, nb)
    b_vals[rng.random(nb) < 0.05] = 0.0
    b_vals[rng.random(nb) < 0.05] = -0.0
    a_pos = a_pos.astype(np.int32)
    rp, rc, rv = orc.add_csr(n, a_pos, a_crd.astype(np.int32), a_vals, b_cols.astype(np.int32),
                             b_vals, b_rows=b_rows.astype(np.int32))
    pos, crd, vals = K.add_csr(n, cuda(a_pos), cuda(a_crd, np.int32), cuda(a_vals),
                               cuda(b_cols, np.int32), cuda(b_vals),
                               b_rows=cuda(b_rows, np.int32), two_pass=two_pass)
    assert np.array_equal(pos.cpu().numpy(), rp)
    assert np.array_equal(crd.cpu().numpy(), rc)
    assert np.array_equal(bits(vals), bits(rv))


@pytest.mark.slow
def test_add_full_size(orc):
    d = wl.add_ab()
    n = d["nrows"]
    rp, rc, rv = orc.add_csr(n, d["a_pos"], d["a_crd"], d["a_vals"], d["b_cols"], d["b_vals"],
                             b_rows=d["b_rows"], threads=0)
    pos, crd, vals = K.add_csr(n, cuda(d["a_pos"]), cuda(d["a_crd"]), cuda(d["a_vals"]),
                               cuda(d["b_cols"]), cuda(d["b_vals"]), b_rows=cuda(d["b_rows"]))
    assert np.array_equal(pos.cpu().numpy(), rp)
    assert np.array_equal(crd.cpu().numpy(), rc)
    assert np.array_equal(bits(vals), bits(rv))
    # structure property: nnz(C) = nnz(A) + nnz(B) - overlap
    assert int(rp[-1]) == len(d["a_crd"]) + len(d["b_cols"]) - d["overlap"]


# ---------------------------------------------------------------------------
# MTTKRP

def _mttkrp_both(c_or_d, I, J, Kd, coo, csf, B, C):
    Bt, Ct = cuda(B), cuda(C)
    A1 = K.mttkrp_coo3(I, J, Kd, cuda(coo[0]), cuda(coo[1]), cuda(coo[2]), cuda(coo[3]), Bt, Ct)
    A2 = K.mttkrp_csf(I, J, Kd, cuda(csf["crd0"]), cuda(csf["pos1"]), cuda(csf["crd1"]),
                      cuda(csf["pos2"]), cuda(csf["crd2"]), cuda(coo[3]), Bt, Ct)
    return A1.cpu().numpy(), A2.cpu().numpy()


def test_mttkrp_goldens(golden, orc):
    for name, c in golden["mttkrp"].items():
        I, J, Kd = int(c["I"]), int(c["J"]), int(c["K"])
        coo = (c["coo_i"], c["coo_j"], c["coo_k"], c["coo_vals"])
        csf = {f"{k}{l}": c[f"csf_{k}{l}"] for k in ("pos", "crd") for l in range(3)}
        A1, A2 = _mttkrp_both(c, I, J, Kd, coo, csf, c["B"], c["C"])
        _, absA = orc.mttkrp_coo3(I, *coo, c["B"], c["C"])
        ok1, e1 = orc.within_condition(A1, c["A_coo"], absA, RTOL)
        ok2, e2 = orc.within_condition(A2, c["A_csf"], absA, RTOL)
        assert ok1 and ok2, (name, e1, e2)


@pytest.mark.parametrize("I,J,Kd,nnz,R,seed", [
    (2000, 1500, 1000, 400_000, 32, 1), (300, 200, 100, 50_000, 16, 2),
    (50, 40, 30, 20_000, 64, 3), (5000, 100, 100, 3000, 32, 4), (20, 3000, 3000, 200_000, 32, 5),
    (400, 300, 200, 60_000, 8, 6), (100, 90, 80, 30_000, 100, 7), (60, 50, 40, 8_000, 200, 8)])
def test_mttkrp_vs_oracle(orc, I, J, Kd, nnz, R, seed):
    m = wl.mttkrp(I=I, J=J, K=Kd, nnz=nnz, R=R, seed=seed)
    csf = wl.coo3_to_csf(m["i"], m["j"], m["k"], None)
    ref, absA = orc.mttkrp_coo3(I, m["i"], m["j"], m["k"], m["vals"], m["B"], m["C"])
    A1, A2 = _mttkrp_both(None, I, J, Kd, (m["i"], m["j"], m["k"], m["vals"]), csf, m["B"], m["C"])
    for A in (A1, A2):
        ok, err = orc.within_condition(A, ref, absA, RTOL)
        assert ok, err
    # determinism: the chunked reduction has a fixed order
    A1b, A2b = _mttkrp_both(None, I, J, Kd, (m["i"], m["j"], m["k"], m["vals"]), csf, m["B"],
                            m["C"])
    assert np.array_equal(bits(A1), bits(A1b)) and np.array_equal(bits(A2), bits(A2b))


@pytest.mark.slow
def test_mttkrp_full_size(orc):
    m = wl.mttkrp()
    csf = wl.coo3_to_csf(m["i"], m["j"], m["k"], None)
    ref, absA = orc.mttkrp_coo3(m["I"], m["i"], m["j"], m["k"], m["vals"], m["B"], m["C"])
    A1, A2 = _mttkrp_both(None, m["I"], m["J"], m["K"], (m["i"], m["j"], m["k"], m["vals"]), csf,
                          m["B"], m["C"])
    for name, A in (("coo3", A1), ("csf", A2)):
        ok, err = orc.within_condition(A, ref, absA, RTOL)
        assert ok, err
        # also the strict |gpu - ref| <= 1e-12 |ref| pass count,
        # expected to miss only a handful of cancelling components
        A = np.asarray(A.cpu().numpy() if hasattr(A, "cpu") else A).reshape(ref.shape)
        d = np.abs(A - ref)
        strict = d <= RTOL * np.abs(ref)
        frac = float(strict.mean())
        print(f"MTTKRP {name}: strict 1e-12 pass {int(strict.sum())}/{strict.size} ({frac:.6f}); "
              f"max |d|/max(|ref|,sum|terms|) {float((d / np.maximum(np.abs(ref), absA)).max()):.3e}; "
              f"bit-identical {int((A == ref).sum())}")
        assert frac >= 0.999, (name, frac)


# ---------------------------------------------------------------------------
# the persistent TMA pipelines (SL_SPMV_PATH=pipe) must agree bit for bit

@pytest.fixture
def pipe_path(monkeypatch):
    if not K.L().sl_build_features() & 1:
        pytest.skip("the TMA pipelines are an A/B build (SL_BUILD_ALT=1)")
    monkeypatch.setenv("SL_SPMV_PATH", "pipe")
    yield


def test_pipe_path_goldens(golden, pipe_path):
    test_spmv_goldens_all_formats(golden)


@pytest.mark.parametrize("n,nnz,lam,seed", [(3000, 30000, 10.0, 1), (5000, 200, 0.05, 2),
                                            (777, 60000, 77.0, 5)])
def test_pipe_path_vs_oracle(orc, pipe_path, n, nnz, lam, seed):
    test_spmv_coo_csr_vs_oracle(orc, n, nnz, lam, seed)


def test_pipe_path_full_size(orc, pipe_path):
    test_spmv_dia_vs_oracle_odd_shapes(orc)
    s = wl.stencil27()
    ref, _ = orc.spmv_csr(s["nrows"], s["pos"], s["crd"], s["vals"], s["x"])
    x = cuda(s["x"])
    y = K.spmv_csr(s["nrows"], s["ncols"], cuda(s["pos"]), cuda(s["crd"]), cuda(s["vals"]), x)
    assert np.array_equal(bits(y), bits(ref))
    e = wl.csr_to_ell(s["pos"], s["crd"], s["vals"], s["nrows"])
    y = K.spmv_ell(s["nrows"], s["ncols"], e["nslots"], cuda(e["crd"]), cuda(e["vals"]), x)
    assert np.array_equal(bits(y), bits(ref))
    d = wl.coo_spmv()
    ref, _ = orc.spmv_coo(d["nrows"], d["rows"], d["cols"], d["vals"], d["x"])
    y = K.spmv_coo(d["nrows"], d["ncols"], cuda(d["rows"]), cuda(d["cols"]), cuda(d["vals"]),
                   cuda(d["x"]))
    assert np.array_equal(bits(y), bits(ref))


def test_mttkrp_scalar_path_matches(orc, monkeypatch):
    """SL_MTTKRP_SCALAR selects the lane-per-column kernels; same tolerance."""
    monkeypatch.setenv("SL_MTTKRP_SCALAR", "1")
    m = wl.mttkrp(I=700, J=500, K=400, nnz=150_000, R=32, seed=11)
    csf = wl.coo3_to_csf(m["i"], m["j"], m["k"], None)
    ref, absA = orc.mttkrp_coo3(700, m["i"], m["j"], m["k"], m["vals"], m["B"], m["C"])
    A1, A2 = _mttkrp_both(None, 700, 500, 400, (m["i"], m["j"], m["k"], m["vals"]), csf, m["B"],
                          m["C"])
    for A in (A1, A2):
        ok, err = orc.within_condition(A, ref, absA, RTOL)
        assert ok, err


def test_dia_row_block_shards(orc):
    from paper_1804_10112_b200 import dist as D
    g = wl.dia7(g=32)
    n = g["nrows"]
    ref, _ = orc.spmv_dia(n, n, g["offsets"], g["vals"], g["x"])
    x = cuda(g["x"])
    ys = []
    for r0, r1 in ((0, 5000), (5000, 20011), (20011, n)):
        offs, v = D.shard_dia(g["offsets"], g["vals"], n, r0, r1)
        ys.append(K.spmv_dia(r1 - r0, n, offs, cuda(v), x, row0=r0).cpu().numpy())
    assert np.array_equal(bits(np.concatenate(ys)), bits(ref))


def test_mttkrp_heavy_rows_span_many_chunks(orc, monkeypatch):
    """Rows longer than 64 chunks (x 2048 nonzeros) exercise the group prefix."""
    rng = np.random.default_rng(21)
    I, J, Kd, R = 5, 1000, 600, 32
    lens = [300_000, 1, 0, 150_000, 2049]
    i = np.repeat(np.arange(I, dtype=np.int32), lens)
    keys = []
    for r, n in enumerate(lens):
        kk = np.sort(rng.choice(J * Kd, size=n, replace=False))
        keys.append(kk)
    jk = np.concatenate(keys)
    j, k = (jk // Kd).astype(np.int32), (jk % Kd).astype(np.int32)
    vals = 1.0 - rng.random(len(i))
    B, C = rng.uniform(-1, 1, (J, R)), rng.uniform(-1, 1, (Kd, R))
    ref, absA = orc.mttkrp_coo3(I, i, j, k, vals, B, C)
    csf = wl.coo3_to_csf(i, j, k, None)
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("SL_MTTKRP_NOREUSE", env)
        A1, A2 = _mttkrp_both(None, I, J, Kd, (i, j, k, vals), csf, B, C)
        for A in (A1, A2):
            ok, err = orc.within_condition(A, ref, absA, RTOL)
            assert ok, err


# ---------------------------------------------------------------------------
# degenerate shapes: no rows, no columns, no slots / diagonals, all-empty rows

def test_spmv_degenerate_shapes(orc):
    e_i, e_f = cuda(np.zeros(0, np.int32)), cuda(np.zeros(0))
    # zero rows: nothing to write, no error
    y = K.spmv_coo(0, 5, e_i, e_i, e_f, cuda(np.ones(5)))
    assert y.numel() == 0
    for variant in CSR_VARIANTS:
        y = K.spmv_csr(0, 5, cuda(np.zeros(1, np.int32)), e_i, e_f, cuda(np.ones(5)),
                       variant=variant)
        assert y.numel() == 0
    # zero columns: every row empty -> +0.0 everywhere
    n = 1000
    x0 = cuda(np.zeros(0))
    for variant in CSR_VARIANTS:
        y = cuda(np.full(n, np.nan))
        K.spmv_csr(n, 0, cuda(np.zeros(n + 1, np.int32)), e_i, e_f, x0, y=y, variant=variant)
        assert np.array_equal(bits(y), bits(np.zeros(n))), variant
    y = cuda(np.full(n, np.nan))
    K.spmv_coo(n, 0, e_i, e_i, e_f, x0, y)
    assert np.array_equal(bits(y), bits(np.zeros(n)))
    # ELL with zero slots, DIA with zero diagonals
    y = cuda(np.full(n, np.nan))
    K.spmv_ell(n, 7, 0, e_i, e_f, cuda(np.ones(7)), y)
    assert np.array_equal(bits(y), bits(np.zeros(n)))
    y = cuda(np.full(n, np.nan))
    K.spmv_dia(n, 7, np.zeros(0, np.int32), e_f, cuda(np.ones(7)), y)
    assert np.array_equal(bits(y), bits(np.zeros(n)))
    # DIA whose diagonals are all out of range for some rows (tall matrix)
    offs = np.array([5, 9], np.int32)
    vals = np.random.default_rng(1).uniform(-1, 1, 2 * n)
    xx = np.random.default_rng(2).uniform(-1, 1, 12)
    ref, _ = orc.spmv_dia(n, 12, offs, vals, xx)
    y = cuda(np.full(n, np.nan))
    K.spmv_dia(n, 12, offs, cuda(vals), cuda(xx), y)
    assert np.array_equal(bits(y), bits(ref))
    # COO whose only nonzeros sit in the last row (every earlier row zeroed
    # by the owner of the last row's start)
    rows = np.full(3, n - 1, np.int32)
    cols = np.array([0, 3, 6], np.int32)
    v = np.array([1.5, -2.0, 0.25])
    xs = np.random.default_rng(3).uniform(-1, 1, 7)
    ref, _ = orc.spmv_coo(n, rows, cols, v, xs)
    y = cuda(np.full(n, np.nan))
    K.spmv_coo(n, 7, cuda(rows), cuda(cols), cuda(v), cuda(xs), y)
    assert np.array_equal(bits(y), bits(ref))


def test_mttkrp_degenerate_and_small_rank(orc):
    # no nonzeros: A is all +0.0; ranks 1 and 3 (scalar path); slices with no
    # nonzeros at both ends of I
    for R in (1, 3, 32):
        I, J, Kd = 50, 20, 10
        z = cuda(np.zeros(0, np.int32))
        A = K.mttkrp_coo3(I, J, Kd, z, z, z, cuda(np.zeros(0)), cuda(np.ones((J, R))),
                          cuda(np.ones((Kd, R))))
        assert np.array_equal(bits(A), bits(np.zeros((I, R)))), R
        rng = np.random.default_rng(R)
        nnz = 500
        key = np.unique(rng.integers(5 * J * Kd, 40 * J * Kd, nnz))     # slices 5..39 only
        i = (key // (J * Kd)).astype(np.int32)
        j = ((key // Kd) % J).astype(np.int32)
        k = (key % Kd).astype(np.int32)
        v = 1.0 - rng.random(len(key))
        Bm, Cm = rng.uniform(-1, 1, (J, R)), rng.uniform(-1, 1, (Kd, R))
        ref, absA = orc.mttkrp_coo3(I, i, j, k, v, Bm, Cm)
        A = K.mttkrp_coo3(I, J, Kd, cuda(i), cuda(j), cuda(k), cuda(v), cuda(Bm), cuda(Cm))
        ok, err = orc.within_condition(A.cpu().numpy(), ref, absA, RTOL)
        assert ok, (R, err)
        assert np.array_equal(bits(A.cpu().numpy()[:5]), bits(np.zeros((5, R))))
        assert np.array_equal(bits(A.cpu().numpy()[40:]), bits(np.zeros((10, R))))


@pytest.mark.parametrize("lam,zipf,seed", [(28.0, None, 1), (None, 1.7, 2)])
def test_add_dense_and_power_law_rows(orc, lam, zipf, seed):
    # tiles far beyond the 768-element stage: the grouped path (consecutive
    # row groups that fit) and single oversized rows (global merge)
    rng = np.random.default_rng(seed)
    n, m = 20_000, 40_000

    def rows_of(lens):
        cols = [np.sort(rng.choice(m, int(k), replace=False)) for k in lens]
        pos = np.zeros(n + 1, np.int64)
        pos[1:] = np.cumsum(lens)
        return pos.astype(np.int32), np.concatenate(cols).astype(np.int32)

    if zipf:
        la = np.minimum(rng.zipf(zipf, n) - 1, 3000)
        lb = np.minimum(rng.zipf(zipf, n) - 1, 3000)
    else:
        la, lb = rng.poisson(lam, n), rng.poisson(lam, n)
    a_pos, a_crd = rows_of(la)
    b_pos, b_cols = rows_of(lb)
    # make ~10% of B's coordinates coincide with A's (matches)
    b_rows = np.repeat(np.arange(n, dtype=np.int32), lb)
    a_vals = rng.uniform(-1, 1, len(a_crd))
    b_vals = rng.uniform(-1, 1, len(b_cols))
    rp, rc, rv = orc.add_csr(n, a_pos, a_crd, a_vals, b_cols, b_vals, b_rows=b_rows)
    for two_pass in (False, True):
        pos, crd, vals = K.add_csr(n, cuda(a_pos), cuda(a_crd), cuda(a_vals), cuda(b_cols),
                                   cuda(b_vals), b_rows=cuda(b_rows), two_pass=two_pass)
        assert np.array_equal(pos.cpu().numpy(), rp), two_pass
        assert np.array_equal(crd.cpu().numpy(), rc), two_pass
        assert np.array_equal(bits(vals), bits(rv)), two_pass


@pytest.mark.parametrize("seed", [3, 4])
def test_add_long_rows_with_matches_and_repeats(orc, seed):
    """Rows far beyond the stage whose B part matches A's columns and repeats
    coordinates (runs of up to 4): the block-cooperative merge path, B runs
    summed as Python's sum() (Neumaier), owners reading ahead across thread
    segments."""
    rng = np.random.default_rng(seed)
    n, m = 3000, 50_000
    la = rng.poisson(4, n)
    lb = rng.poisson(4, n)
    long_rows = rng.choice(n, 12, replace=False)
    la[long_rows] = rng.integers(800, 6000, 12)
    lb[long_rows] = rng.integers(800, 6000, 12)
    a_cols, b_cols, b_rows = [], [], []
    for r in range(n):
        ac = np.sort(rng.choice(m, int(la[r]), replace=False))
        share = ac[rng.random(len(ac)) < 0.3] if len(ac) else ac[:0]
        own = rng.choice(m, int(lb[r]), replace=True)
        bc = np.concatenate([share, own])
        reps = rng.integers(1, 5, len(bc)) * (rng.random(len(bc)) < 0.2) + 1
        bc = np.sort(np.repeat(bc, reps))
        a_cols.append(ac)
        b_cols.append(bc)
        b_rows.append(np.full(len(bc), r))
    a_pos = np.concatenate([[0], np.cumsum([len(c) for c in a_cols])]).astype(np.int32)
    a_crd = np.concatenate(a_cols).astype(np.int32)
    b_cols = np.concatenate(b_cols).astype(np.int32)
    b_rows = np.concatenate(b_rows).astype(np.int32)
    a_vals = rng.uniform(-1, 1, len(a_crd))
    b_vals = rng.uniform(-1, 1, len(b_cols))
    rp, rc, rv = orc.add_csr(n, a_pos, a_crd, a_vals, b_cols, b_vals, b_rows=b_rows)
    for two_pass in (False, True):
        pos, crd, vals = K.add_csr(n, cuda(a_pos), cuda(a_crd), cuda(a_vals), cuda(b_cols),
                                   cuda(b_vals), b_rows=cuda(b_rows), two_pass=two_pass)
        assert np.array_equal(pos.cpu().numpy(), rp), two_pass
        assert np.array_equal(crd.cpu().numpy(), rc), two_pass
        assert np.array_equal(bits(vals), bits(rv)), two_pass
