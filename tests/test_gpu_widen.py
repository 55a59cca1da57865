"""GPU parity of the widened patterns: CSR x sparse-vector
(intersection) and SpMM (CSR x dense-2), against the reference's own
evaluate() outputs (tests/golden/widen.npz) and the oracle at larger sizes.
Bar: bit-exact (single ordered sums per output, no contraction)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1804_10112_b200 as sl  # noqa: E402
from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
from conftest import load_cases  # noqa: E402


def cuda(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a).astype(dtype)), device="cuda")


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1).view(np.int64)


def test_widen_goldens_kernels_and_evaluate():
    seen = 0
    for name, c in load_cases("widen").items():
        if name.startswith("t3"):
            continue
        n, m = int(c["nrows"]), int(c["ncols"])
        A = F.csr_storage(c["csr_pos"], c["csr_crd"], c["csr_vals"], (n, m))
        if name.startswith("spx"):
            y = K.spmv_csr_spx(n, m, cuda(c["csr_pos"], np.int32), cuda(c["csr_crd"], np.int32),
                               cuda(c["csr_vals"], np.float64), cuda(c["x_crd"], np.int32),
                               cuda(c["x_vals"], np.float64))
            assert np.array_equal(bits(y), bits(c["y"])), name
            x = F.sparse_vector_storage(c["x_crd"], c["x_vals"], m)
            y2 = sl.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x})
            assert np.array_equal(bits(y2.vals), bits(c["y"])), name
        else:
            Kc = int(c["K"])
            Y = K.spmm_csr(n, m, cuda(c["csr_pos"], np.int32), cuda(c["csr_crd"], np.int32),
                           cuda(c["csr_vals"], np.float64), cuda(c["X"], np.float64).view(m, Kc))
            assert np.array_equal(bits(Y), bits(c["Y"])), name
            X = F.dense_storage(np.asarray(c["X"]).reshape(m, Kc))
            for expr in ("Y(i,k) = A(i,j) * X(j,k)", "Y(i,k) = X(j,k) * A(i,j)"):
                Y2 = sl.evaluate(expr, {"A": A, "X": X})
                assert Y2.dims == (n, Kc)
                assert np.array_equal(bits(Y2.vals), bits(c["Y"])), (name, expr)
        seen += 1
    assert seen >= 16


@pytest.mark.parametrize("Kc", [1, 2, 5, 8, 16, 32, 40, 64, 72])
def test_spmm_stencil_vs_oracle(orc, Kc):
    st = wl.stencil27(g=24, seed=4)
    n = st["nrows"]
    rng = np.random.default_rng(Kc)
    X = rng.uniform(-1, 1, (n, Kc))
    ref = orc.spmm_csr(n, Kc, st["pos"], st["crd"], st["vals"], X, threads=0)
    Y = K.spmm_csr(n, n, cuda(st["pos"], np.int32), cuda(st["crd"], np.int32),
                   cuda(st["vals"], np.float64), cuda(X, np.float64))
    assert np.array_equal(bits(Y), bits(ref))


def test_spmm_ragged_rows_vs_oracle(orc):
    """rows from 0 to 300 nonzeros (past every lane-group width)"""
    rng = np.random.default_rng(8)
    n, m, Kc = 700, 900, 12
    lens = rng.integers(0, 300, n)
    lens[::7] = 0
    pos = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=pos[1:])
    crd = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.uniform(-1, 1, len(crd))
    X = rng.uniform(-1, 1, (m, Kc))
    ref = orc.spmm_csr(n, Kc, pos.astype(np.int32), crd, vals, X, threads=0)
    Y = K.spmm_csr(n, m, cuda(pos, np.int32), cuda(crd, np.int32), cuda(vals, np.float64),
                   cuda(X, np.float64))
    assert np.array_equal(bits(Y), bits(ref))


@pytest.mark.parametrize("Kc", [1, 12, 32, 45])
def test_spmm_long_row_split_vs_oracle(orc, Kc):
    """power-law rows (up to ~20k nonzeros, empty rows) through the split path
    (one CTA per row longer than long_min) for several thresholds, and
    through evaluate(), which takes it when a row exceeds 1024 nonzeros"""
    rng = np.random.default_rng(30 + Kc)
    n, m = 3000, 40_000
    lens = np.minimum((rng.pareto(1.1, n) * 20).astype(np.int64), 20_000)
    lens[::11] = 0
    lens[5] = 20_000
    pos = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=pos[1:])
    crd = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.uniform(-1, 1, len(crd))
    X = rng.uniform(-1, 1, (m, Kc))
    ref = orc.spmm_csr(n, Kc, pos.astype(np.int32), crd, vals, X, threads=0)
    args = (cuda(pos, np.int32), cuda(crd, np.int32), cuda(vals, np.float64), cuda(X, np.float64))
    for long_min in (0, 1, 7, 200, 1024, 10**9):
        Y = K.spmm_csr(n, m, *args, long_min=long_min)
        assert np.array_equal(bits(Y), bits(ref)), long_min
    A = F.csr_storage(pos.astype(np.int32), crd, vals, (n, m))
    Y2 = sl.evaluate("Y(i,k) = A(i,j) * X(j,k)", {"A": A, "X": F.dense_storage(X)})
    assert np.array_equal(bits(Y2.vals), bits(ref))


@pytest.mark.parametrize("frac", [0.0, 0.01, 0.3, 1.0])
def test_spmv_spx_vs_oracle(orc, frac):
    d = wl.coo_spmv(n=50_000, nnz=500_000, seed=12)
    n, m = d["nrows"], d["ncols"]
    pos = wl.coo_to_csr_pos(d["rows"], n)
    rng = np.random.default_rng(int(frac * 100))
    keep = np.sort(rng.choice(m, int(m * frac), replace=False)).astype(np.int32)
    xv = rng.uniform(-1, 1, len(keep))
    ref, _ = orc.spmv_csr_spx(n, pos, d["cols"], d["vals"], keep, xv)
    y = K.spmv_csr_spx(n, m, cuda(pos, np.int32), cuda(d["cols"], np.int32),
                       cuda(d["vals"], np.float64), cuda(keep, np.int32), cuda(xv, np.float64))
    assert np.array_equal(bits(y), bits(ref))


# ---------------------------------------------------------------------------
# 3-tensor kernels beyond MTTKRP: TTV, TTM (CSF) and INNERPROD (COO-3)

def _fiber_ij(c):
    pos1 = np.asarray(c["csf_pos1"], np.int64)
    s = np.repeat(np.arange(len(c["csf_crd0"])), np.diff(pos1))
    return np.asarray(c["csf_crd0"])[s], np.asarray(c["csf_crd1"])


def _csf_storage(c, dims):
    return F.csf_storage(c["csf_pos0"], c["csf_crd0"], c["csf_pos1"], c["csf_crd1"], c["csf_pos2"],
                         c["csf_crd2"], c["csf_vals"], dims)


def test_tensor3_goldens_through_evaluate(orc):
    for name, c in load_cases("widen").items():
        if not name.startswith("t3"):
            continue
        I, J, Kd, R = (int(c[k]) for k in ("I", "J", "K", "R"))
        X = _csf_storage(c, (I, J, Kd))
        v = F.dense_storage(c["v"])
        Y = sl.evaluate("Y(i,j) = X(i,j,k) * v(k)", {"X": X, "v": v})
        assert np.array_equal(bits(Y.vals), bits(c["ttv_dense"])), name
        Yc = sl.evaluate("Y(i,j) = X(i,j,k) * v(k)", {"X": X, "v": v}, F.preset("csr"))
        assert np.array_equal(Yc.levels[1].pos.cpu().numpy(), c["ttv_csr_pos"]), name
        assert np.array_equal(Yc.levels[1].crd.cpu().numpy(), c["ttv_csr_crd"]), name
        assert np.array_equal(bits(Yc.vals), bits(c["ttv_csr_vals"])), name
        U = F.dense_storage(np.asarray(c["U"]).reshape(Kd, R))
        Y3 = sl.evaluate("Y(i,j,r) = X(i,j,k) * U(k,r)", {"X": X, "U": U})
        assert Y3.dims == (I, J, R)
        assert np.array_equal(bits(Y3.vals), bits(c["ttm_dense"])), name
        Xc = F.coo3_storage(c["x_i"], c["x_j"], c["x_k"], c["x_vals"], (I, J, Kd))
        Zc = F.coo3_storage(c["z_i"], c["z_j"], c["z_k"], c["z_vals"], (I, J, Kd))
        a = sl.evaluate("a() = X(i,j,k) * Z(i,j,k)", {"X": Xc, "Z": Zc})
        x = {k: c[f"x_{k}"] for k in ("i", "j", "k", "vals")}
        z = {k: c[f"z_{k}"] for k in ("i", "j", "k", "vals")}
        ref, absr = orc.inner_coo3(x, z)
        assert ref == float(c["inner"][0])
        got = float(a.vals.cpu().numpy()[0])
        assert abs(got - ref) <= 1e-12 * max(abs(ref), absr), (name, got, ref)


def test_tensor3_full_vs_oracle(orc):
    """D5-shaped (scaled) tensor: TTV/TTM bit-exact, INNERPROD within tolerance."""
    t = wl.mttkrp(I=3000, J=2000, K=1500, nnz=2_000_000, R=16, seed=21)
    I, J, Kd = t["I"], t["J"], t["K"]
    csf = wl.coo3_to_csf(t["i"], t["j"], t["k"], None)
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, Kd)
    U = rng.uniform(-1, 1, (Kd, 16))
    args = (I, J, Kd) + tuple(cuda(csf[k], np.int32) for k in ("crd0", "pos1", "crd1", "pos2",
                                                                "crd2")) + (cuda(t["vals"], np.float64),)
    sums, _ = orc.ttv_csf(csf, t["vals"], v)
    pos1 = np.asarray(csf["pos1"], np.int64)
    s = np.repeat(np.arange(len(csf["crd0"])), np.diff(pos1))
    fi, fj = np.asarray(csf["crd0"])[s].astype(np.int64), np.asarray(csf["crd1"]).astype(np.int64)
    Y = K.ttv_csf(*args, cuda(v, np.float64)).cpu().numpy().reshape(-1)
    ref = np.zeros(I * J)
    ref[fi * J + fj] = sums
    assert np.array_equal(bits(Y), bits(ref))
    pos, crd, vals = K.ttv_csf(*args, cuda(v, np.float64), out="csr")
    assert np.array_equal(bits(vals), bits(sums))
    assert np.array_equal(pos.cpu().numpy(), np.concatenate([[0], np.cumsum(np.bincount(fi, minlength=I))]))
    rows = orc.ttm_csf(csf, t["vals"], U)
    Y3 = K.ttm_csf(*args, cuda(U, np.float64)).cpu().numpy().reshape(I * J, 16)
    assert np.array_equal(bits(Y3[fi * J + fj]), bits(rows))
    for long_min in (0, 2):        # every / most fibres through the SpMM long-row split
        Y4 = K.ttm_csf(*args, cuda(U, np.float64), long_min=long_min).cpu().numpy()
        assert np.array_equal(bits(Y4.reshape(I * J, 16)[fi * J + fj]), bits(rows)), long_min
    # inner product with a perturbed copy of the pattern
    keep = rng.random(len(t["i"])) < 0.5
    z = {"i": t["i"][keep], "j": t["j"][keep], "k": t["k"][keep],
         "vals": rng.uniform(-1, 1, int(keep.sum()))}
    x = {"i": t["i"], "j": t["j"], "k": t["k"], "vals": t["vals"]}
    ref, absr = orc.inner_coo3(x, z)
    a = K.inner_coo3(I, J, Kd, tuple(cuda(x[k], np.int32 if k != "vals" else np.float64)
                                     for k in ("i", "j", "k", "vals")),
                     tuple(cuda(z[k], np.int32 if k != "vals" else np.float64)
                           for k in ("i", "j", "k", "vals")))
    got = float(a.cpu().numpy()[0])
    assert abs(got - ref) <= 1e-12 * max(abs(ref), absr)
    a2 = K.inner_coo3(I, J, Kd, tuple(cuda(x[k], np.int32 if k != "vals" else np.float64)
                                      for k in ("i", "j", "k", "vals")),
                      tuple(cuda(z[k], np.int32 if k != "vals" else np.float64)
                            for k in ("i", "j", "k", "vals")))
    assert float(a2.cpu().numpy()[0]) == got          # deterministic


@pytest.mark.slow
def test_plus3_full_size_properties():
    """3rd-order PLUS at D5 scale (40M nonzeros, power-law fibres), by
    size-independent properties: X + X stores X's coordinates with 0 + (x + x)
    = 2x exactly; X + (empty) is the identity copy 0 + x; X + Z with Z every
    other nonzero of X gives X's structure with 0 + (x + z) on Z's entries."""
    mt = wl.mttkrp()
    I, J, Kd = mt["I"], mt["J"], mt["K"]
    T = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    ti, tj, tk, tv = T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"])
    X = F.coo3_storage(ti, tj, tk, tv, (I, J, Kd))
    expr = "A(i,j,k) = X(i,j,k) + Z(i,j,k)"
    C = sl.evaluate(expr, {"X": X, "Z": X}, F.preset("coo-3"))
    for lv, t in zip(C.levels, (ti, tj, tk)):
        assert torch.equal(lv.crd, t)
    assert torch.equal(C.vals, tv + tv)
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    E0 = F.coo3_storage(e, e, e, torch.empty(0, dtype=torch.float64, device="cuda"), (I, J, Kd))
    C = sl.evaluate(expr, {"X": X, "Z": E0}, F.preset("coo-3"))
    assert torch.equal(C.levels[2].crd, tk) and torch.equal(C.vals, tv)
    Z = F.coo3_storage(ti[::2].contiguous(), tj[::2].contiguous(), tk[::2].contiguous(),
                       (tv[::2] * 0.5).contiguous(), (I, J, Kd))
    C = sl.evaluate(expr, {"X": X, "Z": Z}, F.preset("coo-3"))
    assert torch.equal(C.levels[0].crd, ti) and torch.equal(C.levels[2].crd, tk)
    want = tv.clone()
    want[::2] = tv[::2] + tv[::2] * 0.5
    assert torch.equal(C.vals, want)


@pytest.mark.parametrize("seed", [0, 1])
def test_plus3_long_fibres_all_outputs(seed):
    """3rd-order PLUS with fibres far longer than one k-block (the union's
    rows are (fibre, k-block) pairs, engine._plus3) and short ones beside them,
    into COO-3, CSF and dense-3, against a numpy union of unique coordinates:
    0 + (x + z) where both hold the coordinate, 0 + x / 0 + z otherwise."""
    rng = np.random.default_rng(seed)
    I, J, Kd = 5, 7, 700

    def draw(p_long):
        keys = []
        for f in range(I * J):
            n = rng.integers(300, 600) if rng.random() < p_long else rng.integers(0, 6)
            keys.append(f * Kd + np.sort(rng.choice(Kd, size=int(n), replace=False)))
        k = np.concatenate(keys).astype(np.int64)
        return k, rng.uniform(-1, 1, len(k))

    xk, xv = draw(0.4)
    zk, zv = draw(0.4)
    uk = np.union1d(xk, zk)
    vx = np.zeros(len(uk))
    vz = np.zeros(len(uk))
    inx, inz = np.isin(uk, xk), np.isin(uk, zk)
    vx[inx], vz[inz] = xv, zv
    want = 0.0 + np.where(inx & inz, vx + vz, np.where(inx, vx, vz))
    ui, uj, ukk = uk // (J * Kd), (uk // Kd) % J, uk % Kd

    def st(keys, vals):
        return F.coo3_storage((keys // (J * Kd)).astype(np.int32), ((keys // Kd) % J).astype(np.int32),
                              (keys % Kd).astype(np.int32), vals, (I, J, Kd))

    X, Z = st(xk, xv), st(zk, zv)
    expr = "A(i,j,k) = X(i,j,k) + Z(i,j,k)"
    C = sl.evaluate(expr, {"X": X, "Z": Z}, F.preset("coo-3"))
    for lv, t in zip(C.levels, (ui, uj, ukk)):
        assert np.array_equal(lv.crd.cpu().numpy(), t)
    assert np.array_equal(bits(C.vals), bits(want))
    csf = wl.coo3_to_csf(ui, uj, ukk, None)
    C = sl.evaluate(expr, {"X": X, "Z": Z}, F.preset("csf"))
    assert np.array_equal(C.levels[0].crd.cpu().numpy(), csf["crd0"])
    assert np.array_equal(C.levels[1].pos.cpu().numpy(), csf["pos1"])
    assert np.array_equal(C.levels[1].crd.cpu().numpy(), csf["crd1"])
    assert np.array_equal(C.levels[2].pos.cpu().numpy(), csf["pos2"])
    assert np.array_equal(C.levels[2].crd.cpu().numpy(), csf["crd2"])
    assert np.array_equal(bits(C.vals), bits(want))
    # CSF operands take the same route (fibre keys from the level arrays)
    xc = wl.coo3_to_csf(xk // (J * Kd), (xk // Kd) % J, xk % Kd, None)
    Xc = F.csf_storage(xc["pos0"], xc["crd0"], xc["pos1"], xc["crd1"], xc["pos2"], xc["crd2"],
                       xv, (I, J, Kd))
    D = sl.evaluate(expr, {"X": Xc, "Z": Z}, F.preset("dense", order=3))
    dense = np.zeros(I * J * Kd)
    dense[uk] = want
    assert np.array_equal(bits(D.vals), bits(dense))
