"""GPU: the reference-facing API — device level functions (replaying
pkg/tests/test_levels.py through sl_level_query) and `evaluate` over every
supported pattern, checked against the reference's goldens."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1804_10112_b200 as slb  # noqa: E402
from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import levels as L  # noqa: E402
from paper_1804_10112_b200.errors import (HashSegmentFullError, UnsupportedCapabilityError,  # noqa: E402
                                          UnsupportedMergeError)


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def make_storage(kind):   # test_levels.py:27-40
    E = L.EMPTY
    if kind is L.LevelKind.DENSE:
        return L.LevelStorage(L.dense(), n=4)
    if kind is L.LevelKind.RANGE:
        return L.LevelStorage(L.range_level(), n=4, m=6, offset=[0, -1])
    if kind is L.LevelKind.COMPRESSED:
        return L.LevelStorage(L.compressed(), pos=[0, 2], crd=[0, 1])
    if kind is L.LevelKind.SINGLETON:
        return L.LevelStorage(L.singleton(), crd=[0, 1])
    if kind is L.LevelKind.OFFSET:
        return L.LevelStorage(L.offset_level(), offset=[0, -1], range_n=4)
    return L.LevelStorage(L.hashed(), w=4, crd=[E] * 4)


SUPPORTED = {
    L.LevelKind.DENSE: {"coord_bounds", "coord_access", "locate", "size"},
    L.LevelKind.RANGE: {"coord_bounds", "coord_access"},
    L.LevelKind.COMPRESSED: {"pos_bounds", "pos_access"},
    L.LevelKind.SINGLETON: {"pos_bounds", "pos_access"},
    L.LevelKind.OFFSET: {"pos_bounds", "pos_access"},
    L.LevelKind.HASHED: {"pos_bounds", "pos_access", "locate", "size"},
}
CALLS = {
    "coord_bounds": lambda lv: lv.coord_bounds([0]),
    "coord_access": lambda lv: lv.coord_access(0, [0, 0]),
    "pos_bounds": lambda lv: lv.pos_bounds(0),
    "pos_access": lambda lv: lv.pos_access(0, [0]),
    "locate": lambda lv: lv.locate(0, [0, 0]),
    "size": lambda lv: lv.size(1),
}


@pytest.mark.parametrize("kind", list(L.LevelKind))
@pytest.mark.parametrize("fn", sorted(CALLS))
def test_capability_conformance_device(kind, fn):
    lv = make_storage(kind)
    if fn in SUPPORTED[kind]:
        CALLS[fn](lv)
    else:
        with pytest.raises(UnsupportedCapabilityError):
            CALLS[fn](lv)


def test_level_function_kats(level_kats):
    k = level_kats
    lv = L.LevelStorage(L.range_level(), n=4, m=6, offset=k["range_offsets"])
    lo, hi = lv.query("coord_bounds", np.arange(4))
    assert np.array_equal(np.stack([lo.cpu(), hi.cpu()], 1).reshape(-1), k["range_bounds"])
    q = k["range_access_in"].reshape(-1, 2)
    p, f = lv.query("coord_access", q[:, 0], q[:, 1])
    assert np.array_equal(p.cpu().numpy(), k["range_access_out"]) and f.cpu().numpy().all()
    lv = L.LevelStorage(L.offset_level(), offset=k["range_offsets"], range_n=4)
    q = k["offset_access_in"].reshape(-1, 2)
    c, f = lv.query("pos_access", q[:, 0], q[:, 1])
    assert np.array_equal(c.cpu().numpy(), k["offset_access_out"])
    lv = L.LevelStorage(L.compressed(), pos=k["compressed_pos"], crd=k["compressed_crd"])
    lo, hi = lv.query("pos_bounds", np.arange(4))
    assert np.array_equal(np.stack([lo.cpu(), hi.cpu()], 1).reshape(-1), k["compressed_bounds"])
    c, _ = lv.query("pos_access", np.arange(7))
    assert np.array_equal(c.cpu().numpy(), k["compressed_access"])
    for tag, w in (("h4", 4), ("h8", 8), ("h16", 16)):
        lv = L.LevelStorage(L.hashed(), w=w, crd=k[f"{tag}_crd"])
        p, f = lv.query("locate", np.zeros(len(k[f"{tag}_locate_q"])), k[f"{tag}_locate_q"])
        assert np.array_equal(p.cpu().numpy(), k[f"{tag}_locate_pos"]), tag
        assert np.array_equal(f.cpu().numpy(), k[f"{tag}_locate_found"]), tag
        _, f = lv.query("pos_access", np.arange(w))
        assert np.array_equal(f.cpu().numpy(), k[f"{tag}_pos_found"]), tag
    lv = L.LevelStorage(L.dense(), n=6)
    assert lv.locate(1, [1, 5]) == (int(k["dense_locate_1_5"][0]), True)
    assert lv.coord_access(3, [3, 4]) == (int(k["dense_access_3_4"][0]), True)
    assert lv.size(4) == int(k["dense_size_4"][0])
    # scalar API (test_levels.py:107-122, 146-200)
    assert L.LevelStorage(L.range_level(), n=4, m=6, offset=[0, -1]).coord_bounds([1]) == (1, 4)
    assert L.LevelStorage(L.hashed(), w=4, crd=[L.EMPTY] * 16).pos_bounds(2) == (8, 12)
    assert L.LevelStorage(L.offset_level(), offset=[-2, -1, 0, 1],
                          range_n=4).pos_access(7, [1, 3]) == (2, True)
    lv = L.LevelStorage(L.hashed(), w=4, crd=[L.EMPTY, 1, L.EMPTY, 3])
    assert lv.locate(0, [3]) == (3, True) and lv.locate(0, [2]) == (-1, False)


def test_device_insert_protocol(level_kats):
    lv = L.LevelStorage(L.hashed(), w=4)
    lv.insert_init(1, 4)
    assert lv.crd.cpu().tolist() == [L.EMPTY] * 4
    for c in (3, 2, 6):
        lv.insert_coord(c % 4, c)
    assert lv.crd.cpu().tolist() == level_kats["h4_crd"].tolist()   # one-at-a-time = sequential
    lv.insert_coord(2, 2)  # idempotent
    assert sorted(lv.crd.cpu().tolist()) == sorted(level_kats["h4_crd"].tolist())
    lv = L.LevelStorage(L.hashed(), w=2)
    lv.insert_init(1, 2)
    lv.insert_coord(0, 0)
    lv.insert_coord(0, 2)
    with pytest.raises(HashSegmentFullError):
        lv.insert_coord(0, 4)


def test_append_protocol(level_kats):
    lv = L.LevelStorage(L.compressed())
    lv.append_init(4, 0)
    p = 0
    for row, cols in enumerate([[3, 5], [], [0, 4], [1, 2, 3]]):
        for c in cols:
            lv.append_coord(p, c)
            p += 1
        lv.append_edges(row, p - len(cols), p)
    lv.append_finalize(4, p)
    assert lv.pos.cpu().tolist() == level_kats["append_pos"].tolist()
    assert lv.crd.cpu().tolist() == level_kats["append_crd"].tolist()


def test_evaluate_spmv_all_formats(golden):
    c = golden["spmv"]["spmv_rand2"]
    n, m = int(c["nrows"]), int(c["ncols"])
    x = F.dense_storage(c["x"])
    mats = {
        "coo": F.coo_storage(c["coo_rows"], c["coo_cols"], c["coo_vals"], (n, m)),
        "csr": F.csr_storage(c["csr_pos"], c["csr_crd"], c["csr_vals"], (n, m)),
        "ell": F.ell_storage(int(c["ell_nslots"]), c["ell_crd"], c["ell_vals"], (n, m)),
        "dia": F.dia_storage(c["dia_offsets"], c["dia_vals"], (n, m)),
    }
    for fmt, A in mats.items():
        stats = slb.EvalStats()
        y = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x}, stats=stats)
        assert np.array_equal(bits(y.vals), bits(c[f"{fmt}_y"])), fmt
        assert stats.total() > 0
        # commuted product is bitwise the same
        y2 = slb.evaluate("y(i) = x(j) * A(i,j)", {"A": A, "x": x})
        assert np.array_equal(bits(y2.vals), bits(c[f"{fmt}_y"])), fmt
    hx = F.hash_vector_storage(c["hash_crd"], c["hash_vals"], m, int(c["hash_w"]))
    y = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": mats["csr"], "x": hx})
    assert np.array_equal(bits(y.vals), bits(c["hash_y"]))
    with pytest.raises(UnsupportedMergeError):
        slb.evaluate("y(i) = A(i,j) * x(j)", {"A": mats["coo"], "x": hx})


def test_evaluate_host_inputs_moved_to_device(golden):
    c = golden["spmv"]["spmv_rand3"]
    n, m = int(c["nrows"]), int(c["ncols"])
    A = F.csr_storage(c["csr_pos"], c["csr_crd"], c["csr_vals"], (n, m), device=None)
    x = F.dense_storage(c["x"], device=None)
    assert not A.vals.is_cuda
    y = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x})
    assert y.vals.is_cuda and np.array_equal(bits(y.vals), bits(c["csr_y"]))


def test_evaluate_add_and_mttkrp(golden, orc):
    c = golden["add"]["add_rand1"]
    n, m = int(c["nrows"]), int(c["ncols"])
    A = F.csr_storage(c["a_pos"], c["a_crd"], c["a_vals"], (n, m))
    B = F.coo_storage(c["b_rows"], c["b_cols"], c["b_vals"], (n, m))
    for expr in ("C(i,j) = A(i,j) + B(i,j)", "C(i,j) = B(i,j) + A(i,j)"):
        C = slb.evaluate(expr, {"A": A, "B": B}, F.preset("csr"))
        assert np.array_equal(C.levels[1].pos.cpu().numpy(), c["c_pos"])
        assert np.array_equal(C.levels[1].crd.cpu().numpy(), c["c_crd"])
        assert np.array_equal(bits(C.vals), bits(c["c_vals"]))
    t = golden["mttkrp"]["mttkrp_r32"]
    I, J, Kd, R = (int(t[k]) for k in ("I", "J", "K", "R"))
    X1 = F.coo3_storage(t["coo_i"], t["coo_j"], t["coo_k"], t["coo_vals"], (I, J, Kd))
    X2 = F.csf_storage(t["csf_pos0"], t["csf_crd0"], t["csf_pos1"], t["csf_crd1"], t["csf_pos2"],
                       t["csf_crd2"], t["csf_vals"], (I, J, Kd))
    Bs, Cs = F.dense_storage(t["B"], (J, R)), F.dense_storage(t["C"], (Kd, R))
    _, absA = orc.mttkrp_coo3(I, t["coo_i"], t["coo_j"], t["coo_k"], t["coo_vals"], t["B"], t["C"])
    for X in (X1, X2):
        out = slb.evaluate("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)", {"X": X, "B": Bs, "C": Cs})
        ok, err = orc.within_condition(out.vals.cpu().numpy().reshape(I, R), t["A_coo"], absA)
        assert ok, err


# ---------------------------------------------------------------------------
# SpMV into a hash-vector output (the scatter writer's insert protocol)

def test_evaluate_spmv_hashed_output_goldens():
    import paper_1804_10112_b200 as slb
    from paper_1804_10112_b200 import formats as F
    from paper_1804_10112_b200.errors import HashSegmentFullError
    from conftest import load_cases

    for name, c in load_cases("hashout").items():
        n, m, w = int(c["nrows"]), int(c["ncols"]), int(c["width"])
        x = F.dense_storage(np.asarray(c["x"], np.float64))
        mats = {"coo": F.coo_storage(c["coo_rows"], c["coo_cols"], c["coo_vals"], (n, m)),
                "csr": F.csr_storage(c["csr_pos"], c["csr_crd"], c["csr_vals"], (n, m)),
                "ell": F.ell_storage(int(c["ell_nslots"]), c["ell_crd"], c["ell_vals"], (n, m)),
                "dia": F.dia_storage(c["dia_offsets"], c["dia_vals"], (n, m))}
        yfmt = F.preset("hash-vector", width=w)
        for key, A in mats.items():
            if f"{key}_full" in c:
                with pytest.raises(HashSegmentFullError):
                    slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x}, yfmt)
                continue
            y = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x}, yfmt)
            assert y.levels[0].w == int(c[f"{key}_yw"]), (name, key)
            assert np.array_equal(y.levels[0].crd.cpu().numpy(), c[f"{key}_ycrd"]), (name, key)
            got = y.vals.cpu().numpy().view(np.int64)
            assert np.array_equal(got, np.asarray(c[f"{key}_yvals"], np.float64).view(np.int64)), \
                (name, key)


def test_evaluate_csr_skewed_rows_takes_merge_path(orc):
    # one row far longer than the hand-off stages (a tile far heavier than
    # four stages): evaluate picks the merge-path split (cached per row
    # pointer); results stay bit-exact
    from paper_1804_10112_b200 import engine as E
    rng = np.random.default_rng(4)
    n, m = 5000, 20000
    lens = rng.integers(0, 6, n)
    lens[7] = 10000
    cols = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for k in lens]).astype(np.int32)
    pos = np.zeros(n + 1, np.int32)
    pos[1:] = np.cumsum(lens)
    vals = rng.uniform(-1, 1, len(cols))
    xv = rng.uniform(-1, 1, m)
    A = F.csr_storage(pos, cols, vals, (n, m))
    y = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": F.dense_storage(xv)})
    ref, _ = orc.spmv_csr(n, pos, cols, vals, xv)
    assert np.array_equal(y.vals.cpu().numpy().view(np.int64), ref.view(np.int64))
    assert E._csr_variant(A.levels[1]) == 2
    A2 = F.csr_storage(pos[:8], cols[:pos[7]], vals[:pos[7]], (7, m))
    assert E._csr_variant(A2.levels[1]) == 0


@pytest.mark.parametrize("parts", [2, 3])
def test_device_row_shards_reassemble(parts):
    """dist.row_blocks / shard_storage on the device (what evaluate_sharded
    gives each rank): evaluating every block and concatenating is bit-equal
    to the single-GPU evaluate, for SpMV over CSR / COO / ELL / DIA and MTTKRP
    over COO-3 / CSF."""
    from paper_1804_10112_b200 import dist as D
    from paper_1804_10112_b200 import engine as E
    from paper_1804_10112_b200 import workloads as wl

    d = wl.coo_spmv(n=3000, nnz=40000, seed=5)
    n, m = d["nrows"], d["ncols"]
    pos = wl.coo_to_csr_pos(d["rows"], n)
    e = wl.csr_to_ell(pos, d["cols"], d["vals"], n)
    band = np.abs(d["cols"].astype(np.int64) - d["rows"]) <= 300
    dd = wl.dia_from_coo(d["rows"][band], d["cols"][band], d["vals"][band], n, m)
    x = F.dense_storage(d["x"])
    mats = {"csr": F.csr_storage(pos, d["cols"], d["vals"], (n, m)),
            "coo": F.coo_storage(d["rows"], d["cols"], d["vals"], (n, m)),
            "ell": F.ell_storage(e["nslots"], e["crd"], e["vals"], (n, m)),
            "dia": F.dia_storage(dd["offsets"], dd["vals"], (n, m))}
    for name, A in mats.items():
        full = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x}).vals
        cls = E.format_class(A.format)
        b = D.row_blocks(A, cls, parts, n)
        ys = [slb.evaluate("y(i) = A(i,j) * x(j)",
                           {"A": D.shard_storage(A, cls, b[p], b[p + 1]), "x": x}).vals
              for p in range(parts)]
        assert np.array_equal(bits(torch.cat(ys)), bits(full)), name
    mt = wl.mttkrp(I=300, J=200, K=100, nnz=30000, R=8, seed=6)
    csf = wl.coo3_to_csf(mt["i"], mt["j"], mt["k"], None)
    Bf, Cf = F.dense_storage(mt["B"].reshape(-1), (200, 8)), F.dense_storage(mt["C"].reshape(-1), (100, 8))
    for X in (F.coo3_storage(mt["i"], mt["j"], mt["k"], mt["vals"], (300, 200, 100)),
              F.csf_storage([0, len(csf["crd0"])], csf["crd0"], csf["pos1"], csf["crd1"], csf["pos2"],
                            csf["crd2"], mt["vals"], (300, 200, 100))):
        expr = "A(i,r) = X(i,j,k) * B(j,r) * C(k,r)"
        full = slb.evaluate(expr, {"X": X, "B": Bf, "C": Cf}).vals
        cls = E.format_class(X.format)
        b = D.row_blocks(X, cls, parts, 300)
        As = [slb.evaluate(expr, {"X": D.shard_storage(X, cls, b[p], b[p + 1]), "B": Bf,
                                  "C": Cf}).vals for p in range(parts)]
        # MTTKRP's slice sums are parallel reductions: the blocks cut no slice,
        # so the concatenation equals the whole run's result within its tolerance
        assert np.allclose(torch.cat(As).cpu().numpy(), full.cpu().numpy(), rtol=1e-12, atol=1e-12)
    # world size 1: evaluate_sharded is evaluate
    y1 = D.evaluate_sharded("y(i) = A(i,j) * x(j)", {"A": mats["csr"], "x": x}).vals
    assert np.array_equal(bits(y1), bits(slb.evaluate("y(i) = A(i,j) * x(j)",
                                                      {"A": mats["csr"], "x": x}).vals))


def test_spmv_peers_epilogue_gathers_row_blocks():
    """sl_spmv_csr_peers_f64 (the all-gather fused into the SpMV epilogue),
    with local buffers standing in for the ranks' symmetric-memory buffers:
    every block's rows land in every buffer, bit-equal to the whole SpMV —
    through the register hand-off kernel (short rows) and the fallback
    (rows above its limit: computed into the first buffer, copied)."""
    from paper_1804_10112_b200 import dist as D
    from paper_1804_10112_b200 import kernels as K
    from paper_1804_10112_b200 import workloads as wl

    for lam in (10.0, 60.0):
        d = wl.coo_spmv(n=5000, ncols=6000, nnz=int(5000 * lam), lam=lam, seed=11)
        n, m = d["nrows"], d["ncols"]
        pos = wl.coo_to_csr_pos(d["rows"], n)
        A = F.csr_storage(pos, d["cols"], d["vals"], (n, m))
        x = F.dense_storage(d["x"])
        full = slb.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x}).vals
        world = 3
        bufs = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
                for _ in range(world)]
        b = D.row_blocks(A, "csr", world, n)
        for q in range(world):
            r0, r1 = b[q], b[q + 1]
            Aq = D.shard_storage(A, "csr", r0, r1)
            K.spmv_csr_peers(r1 - r0, m, Aq.levels[1].pos, Aq.levels[1].crd, Aq.vals, x.vals,
                             [t.data_ptr() + 8 * r0 for t in bufs])
        for t in bufs:
            assert np.array_equal(bits(t), bits(full)), lam
