"""Pin the C oracle against golden vectors produced by the reference itself.

CPU only.  The oracle is the checker for every GPU parity test, so it must be
bit-identical to the reference interpreter on every fixture before it is
trusted.
"""

import numpy as np
import pytest

from paper_1804_10112_b200 import workloads as wl
from conftest import load_cases


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def test_spmv_formats_bit_exact(golden, orc):
    n_checked = 0
    for name, c in golden["spmv"].items():
        nrows, ncols, x = int(c["nrows"]), int(c["ncols"]), c["x"]
        if "coo_y" in c:
            y, _ = orc.spmv_coo(nrows, c["coo_rows"], c["coo_cols"], c["coo_vals"], x)
            assert np.array_equal(_bits(y), _bits(c["coo_y"])), name
            ymt = orc.spmv_coo(nrows, c["coo_rows"], c["coo_cols"], c["coo_vals"], x, threads=4)
            assert np.array_equal(_bits(ymt), _bits(c["coo_y"])), name
            n_checked += 1
        if "csr_y" in c:
            y, _ = orc.spmv_csr(nrows, c["csr_pos"], c["csr_crd"], c["csr_vals"], x)
            assert np.array_equal(_bits(y), _bits(c["csr_y"])), name
            assert np.array_equal(_bits(orc.spmv_csr(nrows, c["csr_pos"], c["csr_crd"],
                                                     c["csr_vals"], x, threads=3)),
                                  _bits(c["csr_y"])), name
        if "ell_y" in c:
            y, _ = orc.spmv_ell(nrows, int(c["ell_nslots"]), c["ell_crd"], c["ell_vals"], x)
            assert np.array_equal(_bits(y), _bits(c["ell_y"])), name
            assert np.array_equal(_bits(orc.spmv_ell(nrows, int(c["ell_nslots"]), c["ell_crd"],
                                                     c["ell_vals"], x, threads=3)),
                                  _bits(c["ell_y"])), name
        if "dia_y" in c:
            y, _ = orc.spmv_dia(nrows, ncols, c["dia_offsets"], c["dia_vals"], x)
            assert np.array_equal(_bits(y), _bits(c["dia_y"])), name
            assert np.array_equal(_bits(orc.spmv_dia(nrows, ncols, c["dia_offsets"],
                                                     c["dia_vals"], x, threads=3)),
                                  _bits(c["dia_y"])), name
        if "hash_y" in c:
            y, _ = orc.spmv_csr_hashx(nrows, c["csr_pos"], c["csr_crd"], c["csr_vals"],
                                      int(c["hash_w"]), c["hash_crd"], c["hash_vals"])
            assert np.array_equal(_bits(y), _bits(c["hash_y"])), name
    assert n_checked >= 10


def test_spmv_sum_abs_terms(golden, orc):
    c = golden["spmv"]["spmv_rand1"]
    y, a = orc.spmv_csr(int(c["nrows"]), c["csr_pos"], c["csr_crd"], c["csr_vals"], c["x"])
    ref = np.zeros(int(c["nrows"]))
    r = np.repeat(np.arange(int(c["nrows"])), np.diff(c["csr_pos"]))
    np.add.at(ref, r, np.abs(c["csr_vals"] * c["x"][c["csr_crd"]]))
    assert np.allclose(a, ref, rtol=1e-15, atol=0)
    assert (a >= np.abs(y) - 1e-15).all()


def test_add_bit_exact(golden, orc):
    for name, c in golden["add"].items():
        kw = {}
        if "b_pos" in c:
            kw["b_pos"] = c["b_pos"]
        else:
            kw["b_rows"] = c["b_rows"]
        for threads in (None, 3):
            pos, crd, vals = orc.add_csr(int(c["nrows"]), c["a_pos"], c["a_crd"], c["a_vals"],
                                         c["b_cols"], c["b_vals"], threads=threads, **kw)
            assert np.array_equal(pos, c["c_pos"]), name
            assert np.array_equal(crd, c["c_crd"]), name
            assert np.array_equal(_bits(vals), _bits(c["c_vals"])), name


def test_add_keeps_explicit_zeros(golden):
    c = golden["add"]["add_cancel"]
    assert (c["c_vals"] == 0.0).sum() >= 2
    # signed zeros are normalised by the gather writer's 0.0 + value
    assert not np.signbit(c["c_vals"][c["c_vals"] == 0.0]).any()


def test_mttkrp_bit_exact(golden, orc):
    for name, c in golden["mttkrp"].items():
        I = int(c["I"])
        A, absA = orc.mttkrp_coo3(I, c["coo_i"], c["coo_j"], c["coo_k"], c["coo_vals"],
                                  c["B"], c["C"])
        assert np.array_equal(_bits(A), _bits(c["A_coo"])), name
        assert (absA >= np.abs(A)).all()
        A2, _ = orc.mttkrp_csf(I, c["csf_crd0"], c["csf_pos1"], c["csf_crd1"], c["csf_pos2"],
                               c["csf_crd2"], c["csf_vals"], c["B"], c["C"])
        assert np.array_equal(_bits(A2), _bits(c["A_csf"])), name
        assert np.array_equal(_bits(orc.mttkrp_coo3(I, c["coo_i"], c["coo_j"], c["coo_k"],
                                                    c["coo_vals"], c["B"], c["C"], threads=4)),
                              _bits(c["A_coo"])), name
        assert np.array_equal(_bits(orc.mttkrp_csf(I, c["csf_crd0"], c["csf_pos1"],
                                                   c["csf_crd1"], c["csf_pos2"], c["csf_crd2"],
                                                   c["csf_vals"], c["B"], c["C"], threads=4)),
                              _bits(c["A_csf"])), name


def test_hashed_kats(level_kats, orc):
    k = level_kats
    for tag, w in (("h4", 4), ("h8", 8), ("h16", 16)):
        crd, st = orc.hashed_insert(k[f"{tag}_insert_coords"], w)
        assert st == 0
        assert np.array_equal(crd, k[f"{tag}_crd"]), tag
        pos, found = orc.hashed_locate(k[f"{tag}_locate_q"], w, k[f"{tag}_crd"])
        assert np.array_equal(pos, k[f"{tag}_locate_pos"]), tag
        assert np.array_equal(found.astype(np.int32), k[f"{tag}_locate_found"]), tag
    pos, found = orc.hashed_locate(np.array([7]), 4, k["hfull_crd"])
    assert (int(pos[0]), int(found[0])) == tuple(k["hfull_locate_7"])
    w = int(k["hseg_w"])
    crd, st = orc.hashed_insert(k["hseg_coords"], w, nseg=3, parent=k["hseg_parent"])
    assert st == 0 and np.array_equal(crd, k["hseg_crd"])
    pos, found = orc.hashed_locate(k["hseg_q_coord"], w, k["hseg_crd"], parent=k["hseg_q_parent"])
    assert np.array_equal(pos, k["hseg_q_pos"])
    assert np.array_equal(found.astype(np.int32), k["hseg_q_found"])
    # overflow -> HashSegmentFullError in the reference, status 4 here
    _, st = orc.hashed_insert(np.array([0, 2, 4]), 2)
    assert st == 4 and int(k["overflow_raised"]) == 1


def test_generators_match_reference_layouts(golden, level_kats):
    assert int(level_kats["layouts_checked"]) == 1
    for name in ("dia7_g4", "dia7_g5"):
        c = golden["spmv"][name]
        assert np.array_equal(c["gen_offsets"], c["dia_offsets"])
        assert np.array_equal(_bits(c["gen_vals"]), _bits(c["dia_vals"]))
    for name, c in golden["mttkrp"].items():
        assert np.array_equal(c["gen_i"], c["coo_i"]) and np.array_equal(c["gen_k"], c["coo_k"])
        csf = wl.coo3_to_csf(c["coo_i"], c["coo_j"], c["coo_k"], None)
        for lvl in range(3):
            assert np.array_equal(csf[f"pos{lvl}"], c[f"csf_pos{lvl}"]), (name, lvl)
            assert np.array_equal(csf[f"crd{lvl}"], c[f"csf_crd{lvl}"]), (name, lvl)


@pytest.mark.parametrize("threads", [1, 4])
def test_oracle_mt_equals_st_medium(orc, threads):
    d = wl.coo_spmv(n=5000, nnz=40000, seed=77)
    y1, _ = orc.spmv_coo(5000, d["rows"], d["cols"], d["vals"], d["x"])
    y2 = orc.spmv_coo(5000, d["rows"], d["cols"], d["vals"], d["x"], threads=threads)
    assert np.array_equal(_bits(y1), _bits(y2))
    m = wl.mttkrp(I=200, J=150, K=100, nnz=20000, R=8, seed=78)
    A1, _ = orc.mttkrp_coo3(200, m["i"], m["j"], m["k"], m["vals"], m["B"], m["C"])
    A2 = orc.mttkrp_coo3(200, m["i"], m["j"], m["k"], m["vals"], m["B"], m["C"], threads=threads)
    assert np.array_equal(_bits(A1), _bits(A2))


# ---------------------------------------------------------------------------
# format conversion: the oracle restatement against the reference's convert()

def test_oracle_convert_goldens(orc):
    for name, c in load_cases("convert").items():
        n, m = int(c["nrows"]), int(c["ncols"])
        pos, crd, vals = orc.convert_coo_to_csr(n, c["coo_rows"], c["coo_cols"], c["coo_vals"])
        assert np.array_equal(pos, c["csr_pos"]), name
        assert np.array_equal(crd, c["csr_crd"]), name
        assert orc.bits_equal(vals, c["csr_vals"]), name
        ns, ecrd, evals = orc.convert_csr_to_ell(n, c["csr_pos"], c["csr_crd"], c["csr_vals"])
        assert ns == int(c["ell_nslots"]), name
        assert np.array_equal(ecrd, c["ell_crd"]), name
        assert orc.bits_equal(evals, c["ell_vals"]), name
        if "dia_offsets" in c:
            offs, dv = orc.convert_coo_to_dia(n, m, c["coo_rows"], c["coo_cols"], c["coo_vals"])
            assert np.array_equal(offs, c["dia_offsets"]), name
            assert orc.bits_equal(dv, c["dia_vals"]), name


# ---------------------------------------------------------------------------
# widening: CSR x sparse-vector and SpMM against the reference's evaluate()

def test_oracle_widen_goldens(orc):
    n_spx = n_spmm = 0
    for name, c in load_cases("widen").items():
        if name.startswith("t3"):
            continue
        n = int(c["nrows"])
        if name.startswith("spx"):
            y, _ = orc.spmv_csr_spx(n, c["csr_pos"], c["csr_crd"], c["csr_vals"], c["x_crd"],
                                    c["x_vals"])
            assert orc.bits_equal(y, c["y"]), name
            n_spx += 1
        else:
            K = int(c["K"])
            Y, _ = orc.spmm_csr(n, K, c["csr_pos"], c["csr_crd"], c["csr_vals"], c["X"])
            assert orc.bits_equal(Y.reshape(-1), c["Y"]), name
            Ymt = orc.spmm_csr(n, K, c["csr_pos"], c["csr_crd"], c["csr_vals"], c["X"], threads=4)
            assert orc.bits_equal(Ymt.reshape(-1), c["Y"]), name
            n_spmm += 1
    assert n_spx >= 4 and n_spmm >= 12


def _csf(c):
    return {k: c[f"csf_{k}"] for k in ("pos0", "crd0", "pos1", "crd1", "pos2", "crd2")}


def fiber_coords(c):
    """(i, j) of every CSF fiber"""
    pos1 = np.asarray(c["csf_pos1"], np.int64)
    slice_of = np.repeat(np.arange(len(c["csf_crd0"])), np.diff(pos1))
    return np.asarray(c["csf_crd0"])[slice_of], np.asarray(c["csf_crd1"])


def test_oracle_tensor3_goldens(orc):
    """TTV (dense, CSR), TTM and INNERPROD restatements vs the reference."""
    n = 0
    for name, c in load_cases("widen").items():
        if not name.startswith("t3"):
            continue
        I, J, K, R = (int(c[k]) for k in ("I", "J", "K", "R"))
        fi, fj = fiber_coords(c)
        sums, _ = orc.ttv_csf(_csf(c), c["csf_vals"], c["v"])
        Y = np.zeros(I * J)
        Y[fi * J + fj] = sums
        assert orc.bits_equal(Y, c["ttv_dense"]), name
        assert orc.bits_equal(sums, c["ttv_csr_vals"]), name
        assert np.array_equal(fj, c["ttv_csr_crd"]), name
        counts = np.bincount(fi, minlength=I)
        assert np.array_equal(np.concatenate([[0], np.cumsum(counts)]), c["ttv_csr_pos"]), name
        rows = orc.ttm_csf(_csf(c), c["csf_vals"], np.asarray(c["U"]).reshape(K, R))
        Y3 = np.zeros((I * J, R))
        Y3[fi * J + fj] = rows
        assert orc.bits_equal(Y3.reshape(-1), c["ttm_dense"]), name
        x = {k: c[f"x_{k}"] for k in ("i", "j", "k", "vals")}
        z = {k: c[f"z_{k}"] for k in ("i", "j", "k", "vals")}
        a, _ = orc.inner_coo3(x, z)
        assert orc.bits_equal(np.array([a]), c["inner"]), name
        n += 1
    assert n == 2
