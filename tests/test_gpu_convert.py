"""GPU parity of format conversion (formats.convert, formats.py:583-587;
SURVEY.md §8(f) row 1): against the reference's own convert() outputs
(tests/golden/convert.npz) and the oracle restatement at larger sizes.
Bar: bit-exact structure and values."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1804_10112_b200 as sl  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
from conftest import load_cases  # noqa: E402


def cuda(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a).astype(dtype)), device="cuda")


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def host(t):
    return t.cpu().numpy()


def test_convert_goldens_through_api():
    for name, c in load_cases("convert").items():
        n, m = int(c["nrows"]), int(c["ncols"])
        coo = sl.coo_storage(c["coo_rows"], c["coo_cols"], c["coo_vals"], (n, m))
        csr = sl.convert(coo, sl.preset("csr"))
        assert np.array_equal(host(csr.levels[1].pos), c["csr_pos"]), name
        assert np.array_equal(host(csr.levels[1].crd), c["csr_crd"]), name
        assert np.array_equal(bits(csr.vals), bits(c["csr_vals"])), name
        ell = sl.convert(csr, sl.preset("ell"))
        assert ell.levels[0].n == int(c["ell_nslots"]), name
        assert np.array_equal(host(ell.levels[2].crd), c["ell_crd"]), name
        assert np.array_equal(bits(ell.vals), bits(c["ell_vals"])), name
        ell2 = sl.convert(coo, sl.preset("ell"))
        assert np.array_equal(bits(ell2.vals), bits(c["ell_vals"])), name
        if "dia_offsets" in c:
            dia = sl.convert(coo, sl.preset("dia"))
            assert np.array_equal(host(dia.levels[1].offset), c["dia_offsets"]), name
            assert np.array_equal(bits(dia.vals), bits(c["dia_vals"])), name


def test_convert_two_pass_and_fused_agree():
    c = load_cases("convert")["conv_dup1"]
    n = int(c["nrows"])
    args = (n, cuda(c["coo_rows"], np.int32), cuda(c["coo_cols"], np.int32),
            cuda(c["coo_vals"], np.float64))
    p1, c1, v1 = K.coo_to_csr(*args, path="add", two_pass=True)
    p2, c2, v2 = K.coo_to_csr(*args, path="add", two_pass=False)
    p3, c3, v3 = K.coo_to_csr(*args)        # exact path: repeated coordinates -> A+B passes
    assert torch.equal(p1, p2) and torch.equal(c1, c2) and torch.equal(p1, p3)
    assert torch.equal(c1, c3)
    assert np.array_equal(bits(v1), bits(v2)) and np.array_equal(bits(v1), bits(v3))


@pytest.mark.parametrize("n,nnz,empty_rows", [(20000, 200000, False), (5000, 7, True),
                                             (3000, 29999, True)])
def test_convert_exact_fast_path_unique(orc, n, nnz, empty_rows):
    # unique coordinates: the single streaming pass (row pointer, cols, 0.0 + v);
    # signed zeros in the values, empty rows including leading/trailing ones
    rng = np.random.default_rng(n + nnz)
    m = 4000
    key = np.unique(rng.integers(0, n * m, nnz * 2))[:nnz]
    if empty_rows:
        key = key[(key // m) % 3 != 0]
    r, c = (key // m).astype(np.int32), (key % m).astype(np.int32)
    v = rng.uniform(-1, 1, len(key))
    v[rng.random(len(key)) < 0.05] = -0.0
    pos, crd, vals = K.coo_to_csr(n, cuda(r, np.int32), cuda(c, np.int32), cuda(v, np.float64))
    opos, ocrd, ovals = orc.convert_coo_to_csr(n, r, c, v)
    assert np.array_equal(host(pos), opos) and np.array_equal(host(crd), ocrd)
    assert np.array_equal(bits(vals), bits(ovals))
    # misaligned views take the scalar path of the same pass
    r2 = cuda(np.concatenate([[0], r]), np.int32)[1:]
    c2 = cuda(np.concatenate([[0], c]), np.int32)[1:]
    pos2, crd2, vals2 = K.coo_to_csr(n, r2, c2, cuda(v, np.float64))
    assert np.array_equal(host(pos2), opos) and np.array_equal(host(crd2), ocrd)
    assert np.array_equal(bits(vals2), bits(ovals))


@pytest.mark.parametrize("seed", [0, 1])
def test_convert_vs_oracle_random(orc, seed):
    rng = np.random.default_rng(seed)
    n, m, nnz = 20000 + seed * 777, 15000, 200000
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, m, nnz)
    v = rng.uniform(-1, 1, nnz)
    v[rng.random(nnz) < 0.05] = 0.0
    v[rng.random(nnz) < 0.02] = -0.0
    o = np.lexsort((c, r))
    r, c, v = r[o].astype(np.int32), c[o].astype(np.int32), v[o]
    pos, crd, vals = K.coo_to_csr(n, cuda(r, np.int32), cuda(c, np.int32), cuda(v, np.float64))
    opos, ocrd, ovals = orc.convert_coo_to_csr(n, r, c, v)
    assert np.array_equal(host(pos), opos) and np.array_equal(host(crd), ocrd)
    assert np.array_equal(bits(vals), bits(ovals))
    ns, ecrd, evals = K.csr_to_ell(n, pos, crd, vals)
    ons, oecrd, oevals = orc.convert_csr_to_ell(n, opos, ocrd, ovals)
    assert ns == ons
    assert np.array_equal(host(ecrd), oecrd) and np.array_equal(bits(evals), bits(oevals))
    # unique coordinates for DIA (band matrix so the diagonal count stays small)
    key = np.unique(r.astype(np.int64) * m + np.clip(r + rng.integers(-40, 40, nnz), 0, m - 1))
    ur, uc = (key // m).astype(np.int32), (key % m).astype(np.int32)
    uv = rng.uniform(-1, 1, len(key))
    uv[rng.random(len(key)) < 0.05] = 0.0
    offs, dv = K.coo_to_dia(n, m, cuda(ur, np.int32), cuda(uc, np.int32), cuda(uv, np.float64))
    ooffs, odv = orc.convert_coo_to_dia(n, m, ur, uc, uv)
    assert np.array_equal(host(offs), ooffs)
    assert np.array_equal(bits(dv), bits(odv))


def test_convert_stencil_full_size_properties():
    """64^3 27-point stencil (BASELINE configs[1]): COO -> CSR reproduces the
    generator's CSR, CSR -> ELL its ELL, and convert + CSR SpMV equals the
    direct COO SpMV bit for bit."""
    st = wl.stencil27(g=64, seed=1)
    n = st["nrows"]
    rows = np.repeat(np.arange(n, dtype=np.int32), np.diff(st["pos"]))
    dr, dc, dv = cuda(rows, np.int32), cuda(st["crd"], np.int32), cuda(st["vals"], np.float64)
    pos, crd, vals = K.coo_to_csr(n, dr, dc, dv)
    assert np.array_equal(host(pos), st["pos"]) and np.array_equal(host(crd), st["crd"])
    assert np.array_equal(bits(vals), bits(0.0 + st["vals"]))
    assert np.array_equal(host(K.coo_rowptr(n, dr)), st["pos"])
    ns, ecrd, evals = K.csr_to_ell(n, pos, crd, vals)
    ref = wl.csr_to_ell(st["pos"], st["crd"], 0.0 + st["vals"], n)
    assert ns == ref["nslots"]
    assert np.array_equal(host(ecrd), ref["crd"]) and np.array_equal(bits(evals), bits(ref["vals"]))
    x = cuda(st["x"], np.float64)
    y_coo = K.spmv_coo(n, st["ncols"], dr, dc, dv, x)
    y_csr = K.spmv_csr(n, st["ncols"], pos, crd, vals, x)
    assert np.array_equal(bits(y_coo), bits(y_csr))


def test_convert_dia7_full_size():
    d = wl.dia7(g=64, seed=3)
    n, m = d["nrows"], d["ncols"]
    # expand the generator's DIA to COO on the host, convert back on the device
    offs = np.asarray(d["offsets"], dtype=np.int64)
    dv = np.asarray(d["vals"]).reshape(len(offs), n)
    r = np.arange(n)
    rr, cc, vv = [], [], []
    for k, o in enumerate(offs):
        ok = (r + o >= 0) & (r + o < m) & (dv[k] != 0.0)
        rr.append(r[ok]); cc.append(r[ok] + o); vv.append(dv[k][ok])
    rr, cc, vv = np.concatenate(rr), np.concatenate(cc), np.concatenate(vv)
    o = np.lexsort((cc, rr))
    got_offs, got_vals = K.coo_to_dia(n, m, cuda(rr[o], np.int32), cuda(cc[o], np.int32),
                                      cuda(vv[o], np.float64))
    assert np.array_equal(host(got_offs), offs.astype(np.int32))
    want = np.where(np.asarray(d["vals"]) != 0.0, 0.0 + np.asarray(d["vals"]), 0.0)
    assert np.array_equal(bits(got_vals), bits(want))


def test_convert_unsupported_pair():
    st = sl.csr_storage(np.array([0, 1], np.int32), np.array([0], np.int32), np.array([1.0]), (1, 1))
    with pytest.raises(sl.UnsupportedOutputError):
        sl.convert(st, sl.preset("dia"))


# ---------------------------------------------------------------------------
# general gather-append outputs: A + B over CSR/COO operands into CSR or COO,
# and convert CSR -> COO, against the reference's evaluate()/convert()

def _storage(c, tag, fmt, dims):
    if fmt == "csr":
        return sl.csr_storage(c[f"{tag}_pos"], c[f"{tag}_crd"], c[f"{tag}_vals"], dims)
    return sl.coo_storage(c[f"{tag}_rows"], c[f"{tag}_cols"], c[f"{tag}_vals"], dims)


def test_add_any_operands_any_output():
    for name, c in load_cases("addx").items():
        n, m = int(c["nrows"]), int(c["ncols"])
        fa, fb = str(c["fa"]), str(c["fb"])
        A, B = _storage(c, "a", fa, (n, m)), _storage(c, "b", fb, (n, m))
        for expr in ("C(i,j) = A(i,j) + B(i,j)", "C(i,j) = B(i,j) + A(i,j)"):
            C = sl.evaluate(expr, {"A": A, "B": B}, sl.preset("csr"))
            assert np.array_equal(host(C.levels[1].pos), c["c_csr_pos"]), (name, expr)
            assert np.array_equal(host(C.levels[1].crd), c["c_csr_crd"]), (name, expr)
            assert np.array_equal(bits(C.vals), bits(c["c_csr_vals"])), (name, expr)
            Co = sl.evaluate(expr, {"A": A, "B": B}, sl.preset("coo-soa"))
            assert np.array_equal(host(Co.levels[0].crd), c["c_coo_rows"]), (name, expr)
            assert np.array_equal(host(Co.levels[1].crd), c["c_coo_cols"]), (name, expr)
            assert np.array_equal(bits(Co.vals), bits(c["c_coo_vals"])), (name, expr)
        if fa == "csr":
            coo = sl.convert(A, sl.preset("coo-soa"))
            assert np.array_equal(host(coo.levels[0].crd), c["a_to_coo_rows"]), name
            assert np.array_equal(host(coo.levels[1].crd), c["a_to_coo_cols"]), name
            assert np.array_equal(bits(coo.vals), bits(c["a_to_coo_vals"])), name


def test_assemble_on_device_then_evaluate(orc, tmp_path):
    """io -> assemble (device) -> evaluate: the files-to-result path."""
    from paper_1804_10112_b200 import io as IO
    d = wl.coo_spmv(n=3000, nnz=30000, seed=5)
    data = sl.CoordList((3000, 3000), np.stack([d["rows"], d["cols"]], 1), d["vals"])
    IO.write_mtx(data, str(tmp_path / "a.mtx"))
    back = IO.read_mtx(str(tmp_path / "a.mtx"))
    x = sl.dense_storage(d["x"])
    ref, _ = orc.spmv_coo(3000, d["rows"], d["cols"], d["vals"], d["x"])
    for fmt in ("coo-soa", "csr", "ell", "dia"):
        A = sl.assemble(fmt, (3000, 3000), back)
        y = sl.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x})
        assert np.array_equal(bits(y.vals), bits(ref)), fmt
