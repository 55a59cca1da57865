"""Generate golden vectors by running the REFERENCE implementation.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference (`sparselevels`, pure Python) lives read-only under
/root/reference/pkg/src and exists only in the build container, so its
outputs are frozen here as small .npz fixtures that travel with the repo.
Every tensor is assembled by the reference's own `formats.assemble`
(formats.py:361-501) from a seeded coordinate list, evaluated with the
reference's `engine.evaluate` (engine.py:739-764), and both the storage
arrays and the outputs are saved.  The same script checks that the repo's
numpy generators (paper_1804_10112_b200.workloads) lay out storage exactly
as `assemble` does, and records the level-function known-answer tests of
pkg/tests/test_levels.py as explicit (input, output) tables.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import sparselevels as sl  # noqa: E402  (the reference)
from sparselevels import formats as rf  # noqa: E402
from sparselevels import levels as rl  # noqa: E402

from paper_1804_10112_b200 import workloads as wl  # noqa: E402


def coordlist(dims, coords, vals, canonical=False):
    return sl.CoordList(tuple(dims), [(tuple(int(c) for c in cs), float(v))
                                      for cs, v in zip(coords, vals)], canonical=canonical)


def dense_vec(values):
    n = len(values)
    fmt = sl.preset("dense", 1)
    lv = rl.LevelStorage(fmt.levels[0], n=n)
    return sl.TensorStorage(fmt, (n,), [lv], [float(v) for v in values])


def dense_mat(M):
    M = np.asarray(M, dtype=np.float64)
    fmt = sl.preset("dense-2")
    l0 = rl.LevelStorage(fmt.levels[0], n=M.shape[0])
    l1 = rl.LevelStorage(fmt.levels[1], n=M.shape[1])
    return sl.TensorStorage(fmt, M.shape, [l0, l1], M.reshape(-1).tolist())


def i32(a):
    return np.asarray(list(a), dtype=np.int32)


def f64(a):
    return np.asarray(list(a), dtype=np.float64)


# ---------------------------------------------------------------------------
# SpMV family

def spmv_case(name, nrows, ncols, rows, cols, vals, x, hash_width=None, hash_keep=None):
    """Assemble A as COO/CSR/ELL/DIA (+ x as hash vector), evaluate y = A x."""
    out = {"nrows": nrows, "ncols": ncols, "x": f64(x)}
    data = coordlist((nrows, ncols), zip(rows, cols), vals)
    xs = dense_vec(x)
    expr = "y(i) = A(i,j) * x(j)"
    # COO-SoA keeps duplicates and explicit zeros (non-unique level: no canonicalize)
    coo = sl.assemble(sl.preset("coo-soa"), (nrows, ncols), data)
    out["coo_rows"] = i32(coo.levels[0].crd)
    out["coo_cols"] = i32(coo.levels[1].crd)
    out["coo_vals"] = f64(coo.vals[:len(coo.levels[1].crd)] if coo.levels[1].crd else [])
    out["coo_y"] = f64(sl.evaluate(expr, {"A": coo, "x": xs}).vals[:nrows])
    for fmt in ("csr", "ell", "dia"):
        st = sl.assemble(sl.preset(fmt), (nrows, ncols), data)
        if fmt == "csr":
            out["csr_pos"] = i32(st.levels[1].pos)
            out["csr_crd"] = i32(st.levels[1].crd)
            out["csr_vals"] = f64(st.vals[:len(st.levels[1].crd)] if st.levels[1].crd else [])
        elif fmt == "ell":
            out["ell_nslots"] = st.levels[0].n
            out["ell_crd"] = i32(st.levels[2].crd)
            out["ell_vals"] = f64(st.vals[:st.levels[0].n * nrows] if st.levels[0].n else [])
        else:
            out["dia_offsets"] = i32(st.levels[1].offset)
            nd = len(st.levels[1].offset)
            out["dia_vals"] = f64(st.vals[:nd * nrows] if nd else [])
        out[f"{fmt}_y"] = f64(sl.evaluate(expr, {"A": st, "x": xs}).vals[:nrows])
    if hash_width is not None:
        keep = np.asarray(hash_keep, dtype=np.int64)
        hx = sl.assemble(sl.preset("hash-vector", width=hash_width), (ncols,),
                         coordlist((ncols,), [(int(c),) for c in keep], [x[c] for c in keep]))
        csr = sl.assemble(sl.preset("csr"), (nrows, ncols), data)
        out["hash_w"] = hash_width
        out["hash_crd"] = i32(hx.levels[0].crd)
        out["hash_vals"] = f64(hx.vals)
        out["hash_y"] = f64(sl.evaluate(expr, {"A": csr, "x": hx}).vals[:nrows])
    return name, out


def spmv_cases():
    cases = []
    for seed in range(6):
        d = wl.coo_spmv(n=40 + 7 * seed, ncols=50 + 3 * seed, nnz=6 * (40 + 7 * seed), lam=6.0,
                        seed=100 + seed)
        rng = np.random.default_rng(500 + seed)
        keep = np.sort(rng.choice(d["ncols"], size=d["ncols"] // 2, replace=False))
        cases.append(spmv_case(f"spmv_rand{seed}", d["nrows"], d["ncols"], d["rows"], d["cols"],
                               d["vals"], d["x"], hash_width=[64, 32, 128, 32, 256, 64][seed],
                               hash_keep=keep))
    # empty matrix
    cases.append(spmv_case("spmv_empty", 7, 5, [], [], [], np.linspace(-1, 1, 5),
                           hash_width=8, hash_keep=[1, 3]))
    # hypersparse: empty rows at the front, middle and end; single-entry rows
    rows = [3, 3, 9, 17, 17, 17]
    cols = [0, 11, 5, 2, 3, 15]
    rng = np.random.default_rng(7)
    cases.append(spmv_case("spmv_hypersparse", 25, 16, rows, cols, rng.uniform(-1, 1, 6),
                           rng.uniform(-1, 1, 16), hash_width=8, hash_keep=[0, 2, 3, 5, 11]))
    # signed zeros, cancellation, infinities in x would poison: keep finite
    rows = [0, 0, 1, 1, 2, 2, 2, 3]
    cols = [0, 1, 0, 2, 0, 1, 2, 3]
    vals = [-0.0, 1.5, 2.0, -2.0, -0.0, -0.0, -0.0, 1e-300]
    x = [-0.0, 2.0, 1.0, 1e-300]
    cases.append(spmv_case("spmv_signed_zero", 5, 4, rows, cols, vals, x, hash_width=4,
                           hash_keep=[0, 1, 2, 3]))
    # single column / single row
    cases.append(spmv_case("spmv_one_col", 6, 1, [0, 2, 5], [0, 0, 0], [1.0, -2.0, 3.5], [0.25],
                           hash_width=4, hash_keep=[0]))
    cases.append(spmv_case("spmv_one_row", 1, 9, [0] * 5, [0, 2, 4, 6, 8],
                           [1.0, 1e16, -1e16, 3.0, -1.0], np.arange(9, dtype=float) + 1.0,
                           hash_width=16, hash_keep=[0, 2, 4, 6, 8]))
    # stencils, small grids
    st = wl.stencil27(g=4, seed=11)
    r = np.repeat(np.arange(st["nrows"]), np.diff(st["pos"]))
    cases.append(spmv_case("spmv_stencil27_g4", st["nrows"], st["ncols"], r, st["crd"],
                           st["vals"], st["x"]))
    return cases


def coo_duplicates_case():
    """COO with duplicate (i,j) entries: every stored entry is one scatter."""
    rows = [0, 0, 0, 2, 2]
    cols = [1, 1, 3, 0, 0]
    vals = [0.5, 0.25, -1.0, 1e-17, 1.0]
    x = [1.0, 3.0, 5.0, 7.0]
    coo = sl.assemble(sl.preset("coo-soa"), (3, 4), coordlist((3, 4), zip(rows, cols), vals))
    y = sl.evaluate("y(i) = A(i,j) * x(j)", {"A": coo, "x": dense_vec(x)})
    return "spmv_coo_dups", {
        "nrows": 3, "ncols": 4, "x": f64(x),
        "coo_rows": i32(coo.levels[0].crd), "coo_cols": i32(coo.levels[1].crd),
        "coo_vals": f64(coo.vals), "coo_y": f64(y.vals)}


def dia_case(g, seed):
    d = wl.dia7(g=g, seed=seed)
    n = d["nrows"]
    offs = d["offsets"]
    vals = d["vals"].reshape(len(offs), n)
    rows, cols, vv = [], [], []
    for di, off in enumerate(offs.tolist()):
        for i in range(n):
            j = i + off
            if 0 <= j < n and vals[di, i] != 0.0:
                rows.append(i)
                cols.append(j)
                vv.append(vals[di, i])
    st = sl.assemble(sl.preset("dia"), (n, n), coordlist((n, n), zip(rows, cols), vv))
    y = sl.evaluate("y(i) = A(i,j) * x(j)", {"A": st, "x": dense_vec(d["x"])})
    return f"dia7_g{g}", {
        "nrows": n, "ncols": n, "x": d["x"], "dia_offsets": i32(st.levels[1].offset),
        "dia_vals": f64(st.vals), "dia_y": f64(y.vals),
        "gen_offsets": offs, "gen_vals": d["vals"]}


# ---------------------------------------------------------------------------
# A + B

def add_case(name, nrows, ncols, a_rows, a_cols, a_vals, b_rows, b_cols, b_vals, b_fmt="coo-soa"):
    A = sl.assemble(sl.preset("csr"), (nrows, ncols),
                    coordlist((nrows, ncols), zip(a_rows, a_cols), a_vals))
    B = sl.assemble(sl.preset(b_fmt), (nrows, ncols),
                    coordlist((nrows, ncols), zip(b_rows, b_cols), b_vals))
    C = sl.evaluate("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B}, sl.preset("csr"))
    out = {"nrows": nrows, "ncols": ncols,
           "a_pos": i32(A.levels[1].pos), "a_crd": i32(A.levels[1].crd),
           "a_vals": f64(A.vals[:len(A.levels[1].crd)] if A.levels[1].crd else []),
           "c_pos": i32(C.levels[1].pos), "c_crd": i32(C.levels[1].crd), "c_vals": f64(C.vals)}
    if b_fmt == "csr":
        out["b_pos"] = i32(B.levels[1].pos)
        out["b_cols"] = i32(B.levels[1].crd)
        out["b_vals"] = f64(B.vals[:len(B.levels[1].crd)] if B.levels[1].crd else [])
    else:
        out["b_rows"] = i32(B.levels[0].crd)
        out["b_cols"] = i32(B.levels[1].crd)
        out["b_vals"] = f64(B.vals[:len(B.levels[1].crd)] if B.levels[1].crd else [])
    return name, out


def add_cases():
    cases = []
    for seed in range(5):
        n = 30 + 5 * seed
        d = wl.add_ab(n=n, ncols=40, nnz_a=4 * n, nnz_b=4 * n, lam=4.0, overlap=0.3,
                      seed=200 + seed)
        ar = np.repeat(np.arange(n), np.diff(d["a_pos"]))
        cases.append(add_case(f"add_rand{seed}", n, 40, ar, d["a_crd"], d["a_vals"],
                              d["b_rows"], d["b_cols"], d["b_vals"]))
        if seed == 0:
            # same operands, B stored as CSR
            cases.append(add_case("add_rand0_csr", n, 40, ar, d["a_crd"], d["a_vals"],
                                  d["b_rows"], d["b_cols"], d["b_vals"], b_fmt="csr"))
    # cancellation -> explicit zeros; signed zeros; empty rows
    cases.append(add_case("add_cancel", 4, 5,
                          [0, 0, 1, 3], [1, 3, 0, 4], [1.0, -0.0, 2.5, -0.0],
                          [0, 1, 1, 3], [1, 0, 2, 4], [-1.0, -2.5, 0.25, -0.0]))
    # A empty, B empty
    cases.append(add_case("add_a_empty", 5, 6, [], [], [], [0, 2, 2, 4], [5, 0, 3, 1],
                          [1.0, 2.0, 3.0, -4.0]))
    cases.append(add_case("add_b_empty", 5, 6, [1, 1, 3], [0, 5, 2], [1.5, -2.0, 7.0],
                          [], [], []))
    # B with duplicate coordinates (COO is non-unique): grouped and summed
    cases.append(add_case("add_b_dups", 3, 4, [0, 1], [2, 0], [1.0, 1.0],
                          [0, 0, 0, 1, 1, 2, 2], [2, 2, 3, 1, 1, 0, 0],
                          [0.1, 0.2, 5.0, -0.0, -0.0, 1.0, -1.0]))
    return cases


# ---------------------------------------------------------------------------
# MTTKRP

def mttkrp_case(name, I, J, K, nnz, R, seed):
    d = wl.mttkrp(I=I, J=J, K=K, nnz=nnz, R=R, seed=seed)
    coords = list(zip(d["i"], d["j"], d["k"]))
    data = coordlist((I, J, K), coords, d["vals"])
    Bs, Cs = dense_mat(d["B"]), dense_mat(d["C"])
    expr = "A(i,r) = X(i,j,k) * B(j,r) * C(k,r)"
    out = {"I": I, "J": J, "K": K, "R": R, "B": d["B"], "C": d["C"]}
    coo = sl.assemble(sl.preset("coo-3"), (I, J, K), data)
    out["coo_i"] = i32(coo.levels[0].crd)
    out["coo_j"] = i32(coo.levels[1].crd)
    out["coo_k"] = i32(coo.levels[2].crd)
    out["coo_vals"] = f64(coo.vals)
    out["A_coo"] = f64(sl.evaluate(expr, {"X": coo, "B": Bs, "C": Cs}).vals).reshape(I, R)
    csf = sl.assemble(sl.preset("csf"), (I, J, K), data)
    for lvl in range(3):
        out[f"csf_pos{lvl}"] = i32(csf.levels[lvl].pos)
        out[f"csf_crd{lvl}"] = i32(csf.levels[lvl].crd)
    out["csf_vals"] = f64(csf.vals)
    out["A_csf"] = f64(sl.evaluate(expr, {"X": csf, "B": Bs, "C": Cs}).vals).reshape(I, R)
    out["gen_i"], out["gen_j"], out["gen_k"], out["gen_vals"] = d["i"], d["j"], d["k"], d["vals"]
    return name, out


def mttkrp_cases():
    return [
        mttkrp_case("mttkrp_tiny", 6, 5, 7, 40, 4, 300),
        mttkrp_case("mttkrp_r32", 30, 20, 25, 600, 32, 301),
        mttkrp_case("mttkrp_sparse_slices", 50, 8, 9, 30, 3, 302),
    ]


# ---------------------------------------------------------------------------
# Level-function KATs (pkg/tests/test_levels.py), as explicit tables

# ---------------------------------------------------------------------------
# format conversion (formats.convert -> engine.identity_copy, formats.py:583,
# engine.py:775-779)

def _csr_arrays(st, prefix, out):
    out[f"{prefix}_pos"] = i32(st.levels[1].pos)
    out[f"{prefix}_crd"] = i32(st.levels[1].crd)
    out[f"{prefix}_vals"] = f64(st.vals[:len(st.levels[1].crd)] if st.levels[1].crd else [])


def convert_case(name, nrows, ncols, rows, cols, vals, dia=True):
    """COO -> CSR, CSR -> ELL (and, for unique coordinates, COO -> DIA)
    through the reference's own convert()."""
    out = {"nrows": nrows, "ncols": ncols}
    coo = sl.assemble(sl.preset("coo-soa"), (nrows, ncols),
                      coordlist((nrows, ncols), zip(rows, cols), vals))
    out["coo_rows"] = i32(coo.levels[0].crd)
    out["coo_cols"] = i32(coo.levels[1].crd)
    out["coo_vals"] = f64(coo.vals[:len(coo.levels[1].crd)] if coo.levels[1].crd else [])
    csr = rf.convert(coo, sl.preset("csr"))
    _csr_arrays(csr, "csr", out)
    ell = rf.convert(csr, sl.preset("ell"))
    out["ell_nslots"] = ell.levels[0].n
    out["ell_crd"] = i32(ell.levels[2].crd)
    out["ell_vals"] = f64(ell.vals[:ell.levels[0].n * nrows] if ell.levels[0].n else [])
    if dia:
        d = rf.convert(coo, sl.preset("dia"))
        out["dia_offsets"] = i32(d.levels[1].offset)
        nd = len(d.levels[1].offset)
        out["dia_vals"] = f64(d.vals[:nd * nrows] if nd else [])
    return name, out


def convert_cases():
    cases = []
    for seed in range(4):
        rng = np.random.default_rng(900 + seed)
        n, m = 30 + 5 * seed, 25 + 4 * seed
        nnz = 5 * n
        r = rng.integers(0, n, nnz)
        c = rng.integers(0, m, nnz)
        v = rng.uniform(-1, 1, nnz)
        v[rng.random(nnz) < 0.1] = 0.0          # explicit zeros
        v[rng.random(nnz) < 0.05] = -0.0        # signed zeros
        o = np.lexsort((c, r))
        # duplicates kept in COO (non-unique level) -> summed by the copy
        cases.append(convert_case(f"conv_dup{seed}", n, m, r[o], c[o], v[o], dia=False))
        key = np.unique(r * m + c)
        ur, uc = key // m, key % m
        uv = rng.uniform(-1, 1, len(key))
        uv[rng.random(len(key)) < 0.1] = 0.0
        uv[rng.random(len(key)) < 0.05] = -0.0
        cases.append(convert_case(f"conv_uniq{seed}", n, m, ur, uc, uv))
    cases.append(convert_case("conv_empty", 6, 4, [], [], []))
    cases.append(convert_case("conv_hypersparse", 20, 30, [2, 2, 11, 19], [29, 0, 7, 3],
                              [1.5, -2.0, 0.25, 8.0]))
    cases.append(convert_case("conv_all_zero", 4, 4, [0, 1, 3], [0, 2, 1], [0.0, -0.0, 0.0]))
    st = wl.stencil27(g=3, seed=5)
    rr = np.repeat(np.arange(st["nrows"]), np.diff(st["pos"]))
    cases.append(convert_case("conv_stencil_g3", st["nrows"], st["ncols"], rr, st["crd"],
                              st["vals"]))
    return cases


# ---------------------------------------------------------------------------
# widening: CSR x sparse-vector and SpMM

def spx_case(name, nrows, ncols, rows, cols, vals, x_keep, x_vals):
    out = {"nrows": nrows, "ncols": ncols}
    csr = sl.assemble(sl.preset("csr"), (nrows, ncols), coordlist((nrows, ncols), zip(rows, cols), vals))
    _csr_arrays(csr, "csr", out)
    xs = sl.assemble(sl.preset("sparse-vector"), (ncols,),
                     coordlist((ncols,), [(int(c),) for c in x_keep], x_vals))
    out["x_crd"] = i32(xs.levels[0].crd)
    out["x_vals"] = f64(xs.vals[:len(xs.levels[0].crd)] if xs.levels[0].crd else [])
    out["y"] = f64(sl.evaluate("y(i) = A(i,j) * x(j)", {"A": csr, "x": xs}).vals[:nrows])
    return name, out


def spmm_case(name, nrows, ncols, K, rows, cols, vals, X):
    out = {"nrows": nrows, "ncols": ncols, "K": K}
    csr = sl.assemble(sl.preset("csr"), (nrows, ncols), coordlist((nrows, ncols), zip(rows, cols), vals))
    _csr_arrays(csr, "csr", out)
    X = np.asarray(X, dtype=np.float64).reshape(ncols, K)
    out["X"] = X.reshape(-1)
    Y = sl.evaluate("Y(i,k) = A(i,j) * X(j,k)", {"A": csr, "X": dense_mat(X)})
    out["Y"] = f64(Y.vals[:nrows * K])
    return name, out


def dense_tensor(values, dims):
    fmt = sl.preset("dense", len(dims))
    lv = [rl.LevelStorage(l, n=n) for l, n in zip(fmt.levels, dims)]
    return sl.TensorStorage(fmt, tuple(dims), lv, [float(v) for v in np.asarray(values).reshape(-1)])


def tensor3_case(name, I, J, K, nnz, R, seed, nnz_z):
    """TTV (dense and CSR outputs), TTM (dense) and INNERPROD (scalar) on a
    Zipf-ish 3-tensor, through the reference's evaluate()."""
    d = wl.mttkrp(I=I, J=J, K=K, nnz=nnz, R=R, seed=seed)
    data = coordlist((I, J, K), zip(d["i"], d["j"], d["k"]), d["vals"])
    out = {"I": I, "J": J, "K": K, "R": R}
    csf = sl.assemble(sl.preset("csf"), (I, J, K), data)
    for lvl in range(3):
        out[f"csf_pos{lvl}"] = i32(csf.levels[lvl].pos)
        out[f"csf_crd{lvl}"] = i32(csf.levels[lvl].crd)
    out["csf_vals"] = f64(csf.vals)
    rng = np.random.default_rng(seed + 1)
    v = rng.uniform(-1, 1, K)
    v[::7] = -0.0
    U = rng.uniform(-1, 1, (K, R))
    out["v"], out["U"] = v, U.reshape(-1)
    out["ttv_dense"] = f64(sl.evaluate("Y(i,j) = X(i,j,k) * v(k)",
                                       {"X": csf, "v": dense_tensor(v, (K,))}).vals[:I * J])
    yc = sl.evaluate("Y(i,j) = X(i,j,k) * v(k)", {"X": csf, "v": dense_tensor(v, (K,))},
                     sl.preset("csr"))
    _csr_arrays(yc, "ttv_csr", out)
    out["ttm_dense"] = f64(sl.evaluate("Y(i,j,r) = X(i,j,k) * U(k,r)",
                                       {"X": csf, "U": dense_tensor(U, (K, R))}).vals[:I * J * R])
    # inner product against a second tensor sharing part of the pattern
    z = wl.mttkrp(I=I, J=J, K=K, nnz=nnz_z, R=R, seed=seed + 50)
    zi = np.concatenate([d["i"][::3], z["i"]])
    zj = np.concatenate([d["j"][::3], z["j"]])
    zk = np.concatenate([d["k"][::3], z["k"]])
    key = (zi.astype(np.int64) * J + zj) * K + zk
    key, first = np.unique(key, return_index=True)
    zv = np.random.default_rng(seed + 2).uniform(-1, 1, len(key))
    zi, zj, zk = (key // (J * K)), (key // K) % J, key % K
    Xc = sl.assemble(sl.preset("coo-3"), (I, J, K), data)
    Zc = sl.assemble(sl.preset("coo-3"), (I, J, K),
                     coordlist((I, J, K), zip(zi, zj, zk), zv))
    for tag, T in (("x", Xc), ("z", Zc)):
        out[f"{tag}_i"] = i32(T.levels[0].crd)
        out[f"{tag}_j"] = i32(T.levels[1].crd)
        out[f"{tag}_k"] = i32(T.levels[2].crd)
        out[f"{tag}_vals"] = f64(T.vals[:len(T.levels[2].crd)])
    out["inner"] = f64(sl.evaluate("a() = X(i,j,k) * Z(i,j,k)", {"X": Xc, "Z": Zc}).vals)
    return name, out


def widen_cases():
    cases = []
    for seed in range(3):
        d = wl.coo_spmv(n=30 + 11 * seed, ncols=40 + 5 * seed, nnz=6 * (30 + 11 * seed), lam=6.0,
                        seed=300 + seed)
        rng = np.random.default_rng(700 + seed)
        keep = np.sort(rng.choice(d["ncols"], size=d["ncols"] // 3, replace=False))
        xv = rng.uniform(-1, 1, len(keep))
        xv[::5] = -0.0
        cases.append(spx_case(f"spx_rand{seed}", d["nrows"], d["ncols"], d["rows"], d["cols"],
                              d["vals"], keep, xv))
        for K in (1, 3, 8, 33):
            X = rng.uniform(-1, 1, d["ncols"] * K)
            cases.append(spmm_case(f"spmm_rand{seed}_k{K}", d["nrows"], d["ncols"], K, d["rows"],
                                   d["cols"], d["vals"], X))
    cases.append(spx_case("spx_empty_x", 5, 6, [0, 1, 4], [1, 2, 5], [1.0, 2.0, 3.0], [], []))
    cases.append(spx_case("spx_signed", 3, 4, [0, 0, 1, 2], [0, 3, 1, 2], [-0.0, 1.5, -2.0, 0.0],
                          [0, 1, 3], [2.0, -0.0, 1e-300]))
    cases.append(spmm_case("spmm_empty_rows", 4, 3, 2, [1, 1, 3], [0, 2, 1], [1.0, -1.0, 0.5],
                           np.arange(6, dtype=np.float64) - 2.5))
    cases.append(tensor3_case("t3_small", 9, 11, 13, 300, 3, 41, 200))
    cases.append(tensor3_case("t3_medium", 40, 50, 60, 6000, 8, 42, 3000))
    return cases


# ---------------------------------------------------------------------------
# assembly (formats.assemble) and file readers (io.read_mtx / read_tns)

def _storage_arrays(st, prefix, out):
    for k, lv in enumerate(st.levels):
        for attr in ("pos", "crd", "offset"):
            a = getattr(lv, attr, None)
            if a is not None and len(a):
                out[f"{prefix}_l{k}_{attr}"] = i32(a)
        if getattr(lv, "n", None) is not None:
            out[f"{prefix}_l{k}_n"] = int(lv.n)
        if getattr(lv, "w", None):
            out[f"{prefix}_l{k}_w"] = int(lv.w)
    out[f"{prefix}_vals"] = f64(st.vals)


def assembly_case(name, dims, coords, vals, fmts, **kw):
    out = {"dims": np.array(dims), "coords": np.asarray(coords, np.int64).reshape(-1, len(dims)),
           "vals": f64(vals)}
    data = sl.CoordList(tuple(dims), [(tuple(int(x) for x in c), float(v))
                                      for c, v in zip(out["coords"], out["vals"])])
    for f in fmts:
        st = sl.assemble(sl.preset(f, **kw.get(f, {})) if f in kw else sl.preset(f), tuple(dims),
                         data)
        _storage_arrays(st, f.replace("-", "_"), out)
    return name, out


def assembly_cases():
    cases = []
    rng = np.random.default_rng(77)
    n, m, nnz = 12, 9, 60
    c = np.stack([rng.integers(0, n, nnz), rng.integers(0, m, nnz)], 1)
    v = rng.uniform(-1, 1, nnz)
    v[::9] = 0.0
    v[::11] = -0.0
    c[5] = c[3]                      # explicit duplicates, in file order
    c[40] = c[3]
    cases.append(assembly_case("asm_mat", (n, m), c, v,
                               ["coo-soa", "csr", "ell", "dia", "hash-vector"][:4]))
    cases.append(assembly_case("asm_ell_declared", (n, m), c, v, ["ell"], ell={"slots": 12}))
    vec_c = rng.integers(0, 40, (25, 1))
    cases.append(assembly_case("asm_vec", (40,), vec_c, rng.uniform(-1, 1, 25),
                               ["sparse-vector", "hash-vector", "dense"]))
    t = np.stack([rng.integers(0, 5, 80), rng.integers(0, 6, 80), rng.integers(0, 7, 80)], 1)
    tv = rng.uniform(-1, 1, 80)
    tv[::13] = 0.0
    cases.append(assembly_case("asm_t3", (5, 6, 7), t, tv, ["coo-3", "csf"]))
    cases.append(assembly_case("asm_empty", (4, 5), np.zeros((0, 2), np.int64), [],
                               ["coo-soa", "csr", "ell", "dia"]))
    return cases


def io_cases():
    from sparselevels import io as rio
    import tempfile
    texts = {
        "mtx_real": ("mtx", "%%MatrixMarket matrix coordinate real general\n% c\n3 4 4\n"
                            "1 1 1.5\n3 4 -2\n2 2 0\n1 1 0.25\n"),
        "mtx_pattern": ("mtx", "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n"),
        "mtx_int": ("mtx", "%%MatrixMarket matrix coordinate integer general\n\n2 3 1\n2 3 7\n"),
        "mtx_bad_sym": ("mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n"),
        "mtx_bad_count": ("mtx", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n"),
        "mtx_out_of_range": ("mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n"),
        "mtx_no_header": ("mtx", "2 2 1\n1 1 1\n"),
        "mtx_bad_field": ("mtx", "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n"),
        "tns_basic": ("tns", "# t\n1 1 1 1.0\n2 3 1 -2.5\n1 1 1 0.5\n"),
        "tns_bad_order": ("tns", "1 1 1 1.0\n1 1 2.0\n"),
        "tns_zero_based": ("tns", "0 1 1 1.0\n"),
    }
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, (kind, text) in texts.items():
            path = f"{d}/{name}.{kind}"
            with open(path, "w") as fh:
                fh.write(text)
            rec = {"kind": kind, "text": text}
            try:
                cl = rio.read_mtx(path) if kind == "mtx" else rio.read_tns(path)
                rec["dims"] = np.array(cl.dims)
                rec["coords"] = np.array([c for c, _ in cl.entries], np.int64).reshape(
                    -1, len(cl.dims))
                rec["vals"] = f64([v for _, v in cl.entries])
            except rio.FileFormatError as exc:
                rec["error"] = str(exc).replace(d + "/", "")
            out[name] = rec
    return list(out.items())


# ---------------------------------------------------------------------------
# general gather-append outputs: A + B over any CSR/COO
# operands into CSR or COO-SoA, and convert CSR -> COO

def _coo_arrays(st, prefix, out):
    out[f"{prefix}_rows"] = i32(st.levels[0].crd)
    out[f"{prefix}_cols"] = i32(st.levels[1].crd)
    out[f"{prefix}_vals"] = f64(st.vals[:len(st.levels[1].crd)] if st.levels[1].crd else [])


def addx_case(name, n, m, a, b, fa, fb):
    A = sl.assemble(sl.preset(fa), (n, m), coordlist((n, m), zip(a[0], a[1]), a[2]))
    B = sl.assemble(sl.preset(fb), (n, m), coordlist((n, m), zip(b[0], b[1]), b[2]))
    out = {"nrows": n, "ncols": m, "fa": fa, "fb": fb}
    for tag, T, f in (("a", A, fa), ("b", B, fb)):
        if f == "csr":
            _csr_arrays(T, tag, out)
        else:
            _coo_arrays(T, tag, out)
    Cc = sl.evaluate("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B}, sl.preset("csr"))
    _csr_arrays(Cc, "c_csr", out)
    Co = sl.evaluate("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B}, sl.preset("coo-soa"))
    _coo_arrays(Co, "c_coo", out)
    if fa == "csr":
        _coo_arrays(rf.convert(A, sl.preset("coo-soa")), "a_to_coo", out)
    return name, out


def addx_cases():
    cases = []
    rng = np.random.default_rng(91)
    for seed, (fa, fb) in enumerate((("coo-soa", "coo-soa"), ("csr", "csr"), ("coo-soa", "csr"),
                                      ("csr", "coo-soa"))):
        n, m, k = 25, 20, 120
        a = [np.sort(rng.integers(0, n, k)), rng.integers(0, m, k), rng.uniform(-1, 1, k)]
        b = [np.sort(rng.integers(0, n, k)), rng.integers(0, m, k), rng.uniform(-1, 1, k)]
        for x in (a, b):
            o = np.lexsort((x[1], x[0]))
            x[0], x[1], x[2] = x[0][o], x[1][o], x[2][o]
            x[2][::10] = 0.0
            x[2][::17] = -0.0
        cases.append(addx_case(f"addx_{seed}", n, m, a, b, fa, fb))
    return cases


def level_kats():
    """Run the reference level functions on the test_levels.py fixtures."""
    E = rl.EMPTY
    out = {}
    rng = np.random.default_rng(42)
    # range coord_bounds / coord_access (test_levels.py:107-140)
    lv = rl.LevelStorage(rl.range_level(), n=4, m=6, offset=[-2, -1, 0, 1])
    q = [(d, i) for d in range(4) for i in range(*lv.coord_bounds([d]))]
    out["range_offsets"] = i32([-2, -1, 0, 1])
    out["range_bounds"] = i32([v for d in range(4) for v in lv.coord_bounds([d])])
    out["range_access_in"] = i32([v for t in q for v in t])
    out["range_access_out"] = i32([lv.coord_access(d, [d, i])[0] for d, i in q])
    # offset pos_access (test_levels.py:158-161)
    lv = rl.LevelStorage(rl.offset_level(), offset=[-2, -1, 0, 1], range_n=4)
    pa = [(p, pre) for p in range(16) for pre in range(4)]
    out["offset_access_in"] = i32([v for t in pa for v in t])
    out["offset_access_out"] = i32([lv.pos_access(p, [0, pre])[0] for p, pre in pa])
    # compressed pos_bounds (test_levels.py:146-149)
    lv = rl.LevelStorage(rl.compressed(), pos=[0, 2, 4, 4, 7], crd=[0, 1, 0, 1, 1, 2, 4])
    out["compressed_pos"] = i32(lv.pos)
    out["compressed_crd"] = i32(lv.crd)
    out["compressed_bounds"] = i32([v for p in range(4) for v in lv.pos_bounds(p)])
    out["compressed_access"] = i32([lv.pos_access(p, [])[0] for p in range(7)])
    # hashed: insertion (probe wrap), locate hit/miss, pos_access found flags
    for tag, w, coords in (("h4", 4, [3, 2, 6]), ("h8", 8, [1, 9, 17, 3, 4, 12]),
                           ("h16", 16, list(rng.choice(40, 11, replace=False)))):
        lv = rl.LevelStorage(rl.hashed(), w=w)
        lv.insert_init(1, w)
        for c in coords:
            lv.insert_coord(int(c) % w, int(c))
        out[f"{tag}_insert_coords"] = i32(coords)
        out[f"{tag}_crd"] = i32(lv.crd)
        qs = list(range(0, 45))
        res = [lv.locate(0, [c]) for c in qs]
        out[f"{tag}_locate_q"] = i32(qs)
        out[f"{tag}_locate_pos"] = i32([p for p, _ in res])
        out[f"{tag}_locate_found"] = i32([int(f) for _, f in res])
        out[f"{tag}_pos_found"] = i32([int(lv.pos_access(p, [])[1]) for p in range(w)])
    # full segment, absent coordinate: terminates with a miss (test_levels.py:198-200)
    lv = rl.LevelStorage(rl.hashed(), w=4, crd=[0, 1, 2, 3])
    out["hfull_crd"] = i32([0, 1, 2, 3])
    out["hfull_locate_7"] = i32(list(lv.locate(0, [7])))
    # multi-segment hashed level (parent positions > 0)
    w = 8
    lv = rl.LevelStorage(rl.hashed(), w=w)
    lv.insert_init(3, 3 * w)
    seg_coords = [(0, 5), (0, 13), (1, 5), (2, 7), (2, 15), (2, 23), (1, 21)]
    for pp, c in seg_coords:
        lv.insert_coord(pp * w + c % w, c)
    out["hseg_w"] = np.int32(w)
    out["hseg_parent"] = i32([p for p, _ in seg_coords])
    out["hseg_coords"] = i32([c for _, c in seg_coords])
    out["hseg_crd"] = i32(lv.crd)
    qp = [(p, c) for p in range(3) for c in range(0, 30)]
    res = [lv.locate(p, [c]) for p, c in qp]
    out["hseg_q_parent"] = i32([p for p, _ in qp])
    out["hseg_q_coord"] = i32([c for _, c in qp])
    out["hseg_q_pos"] = i32([p for p, _ in res])
    out["hseg_q_found"] = i32([int(f) for _, f in res])
    # overflow (test_levels.py:237-243)
    lv = rl.LevelStorage(rl.hashed(), w=2)
    lv.insert_init(1, 2)
    lv.insert_coord(0, 0)
    lv.insert_coord(0, 2)
    try:
        lv.insert_coord(0, 4)
        out["overflow_raised"] = np.int32(0)
    except sl.HashSegmentFullError:
        out["overflow_raised"] = np.int32(1)
    # dense locate/size
    lv = rl.LevelStorage(rl.dense(), n=6)
    out["dense_locate_1_5"] = i32([lv.locate(1, [1, 5])[0]])
    out["dense_access_3_4"] = i32([lv.coord_access(3, [3, 4])[0]])
    out["dense_size_4"] = i32([lv.size(4)])
    # append protocol (test_levels.py:256-272)
    lv = rl.LevelStorage(rl.compressed())
    lv.append_init(4, 0)
    per_row = [[3, 5], [], [0, 4], [1, 2, 3]]
    p = 0
    for row, cols in enumerate(per_row):
        for c in cols:
            lv.append_coord(p, c)
            p += 1
        lv.append_edges(row, p - len(cols), p)
    out["append_counts"] = i32([len(r) for r in per_row])
    out["append_pos"] = i32(lv.pos)
    out["append_crd"] = i32(lv.crd)
    return out


# ---------------------------------------------------------------------------

def check_generator_layouts():
    """workloads.* must reproduce assemble()'s layouts (formats.py:361-501)."""
    d = wl.coo_spmv(n=60, ncols=70, nnz=300, lam=5.0, seed=9)
    data = coordlist((60, 70), zip(d["rows"], d["cols"]), d["vals"])
    csr = sl.assemble(sl.preset("csr"), (60, 70), data)
    pos = wl.coo_to_csr_pos(d["rows"], 60)
    assert np.array_equal(pos, i32(csr.levels[1].pos))
    assert np.array_equal(d["cols"], i32(csr.levels[1].crd))
    ell = sl.assemble(sl.preset("ell"), (60, 70), data)
    e = wl.csr_to_ell(pos, d["cols"], d["vals"], 60)
    assert e["nslots"] == ell.levels[0].n
    assert np.array_equal(e["crd"], i32(ell.levels[2].crd))
    assert np.array_equal(e["vals"], f64(ell.vals))
    dia = sl.assemble(sl.preset("dia"), (60, 70), data)
    dd = wl.dia_from_coo(d["rows"], d["cols"], d["vals"], 60, 70)
    assert np.array_equal(dd["offsets"], i32(dia.levels[1].offset))
    assert np.array_equal(dd["vals"], f64(dia.vals))
    m = wl.mttkrp(I=9, J=8, K=7, nnz=60, R=2, seed=3)
    data = coordlist((9, 8, 7), zip(m["i"], m["j"], m["k"]), m["vals"])
    csf = sl.assemble(sl.preset("csf"), (9, 8, 7), data)
    c = wl.coo3_to_csf(m["i"], m["j"], m["k"], (9, 8, 7))
    for lvl in range(3):
        assert np.array_equal(c[f"pos{lvl}"], i32(csf.levels[lvl].pos)), lvl
        assert np.array_equal(c[f"crd{lvl}"], i32(csf.levels[lvl].crd)), lvl
    h = wl.hash_vector(n=50, m=20, width=32, seed=5)
    hx = sl.assemble(sl.preset("hash-vector", width=32), (50,),
                     coordlist((50,), [(int(c),) for c in h["coords"]], h["xvals"]))
    assert np.array_equal(h["crd"], i32(hx.levels[0].crd))
    assert np.array_equal(h["vals"], f64(hx.vals))
    return {"layouts_checked": np.int32(1)}


def hashout_case(name, nrows, ncols, rows, cols, vals, x, width):
    """SpMV into a hash-vector y (the scatter writer's insert protocol,
    engine.py:281-327) for COO / CSR / ELL / DIA operands."""
    out = {"nrows": nrows, "ncols": ncols, "x": f64(x), "width": width}
    data = coordlist((nrows, ncols), zip(rows, cols), vals)
    yfmt = sl.preset("hash-vector", width=width)
    for fmt in ("coo-soa", "csr", "ell", "dia"):
        st = sl.assemble(sl.preset(fmt), (nrows, ncols), data)
        key = fmt.split("-")[0]
        if fmt == "coo-soa":
            out["coo_rows"] = i32(st.levels[0].crd)
            out["coo_cols"] = i32(st.levels[1].crd)
            out["coo_vals"] = f64(st.vals[:len(st.levels[1].crd)] if st.levels[1].crd else [])
        elif fmt == "csr":
            out["csr_pos"] = i32(st.levels[1].pos)
            out["csr_crd"] = i32(st.levels[1].crd)
            out["csr_vals"] = f64(st.vals[:len(st.levels[1].crd)] if st.levels[1].crd else [])
        elif fmt == "ell":
            out["ell_nslots"] = st.levels[0].n
            out["ell_crd"] = i32(st.levels[2].crd)
            out["ell_vals"] = f64(st.vals[:st.levels[0].n * nrows] if st.levels[0].n else [])
        else:
            out["dia_offsets"] = i32(st.levels[1].offset)
            nd = len(st.levels[1].offset)
            out["dia_vals"] = f64(st.vals[:nd * nrows] if nd else [])
        try:
            y = sl.evaluate("y(i) = A(i,j) * x(j)", {"A": st, "x": dense_vec(x)}, yfmt)
        except sl.HashSegmentFullError:
            out[f"{key}_full"] = 1                      # more rows written than slots
            continue
        out[f"{key}_ycrd"] = i32(y.levels[0].crd)
        out[f"{key}_yw"] = y.levels[0].w
        out[f"{key}_yvals"] = f64(y.vals)
    return name, out


def hashout_cases():
    rng = np.random.default_rng(61)
    cases = []
    # small: empty rows, an explicit zero, default width (next_pow2(2n))
    cases.append(hashout_case("ho_small", 8, 6, [0, 0, 2, 2, 5, 6], [1, 3, 0, 2, 4, 1],
                              [2.0, -1.0, 0.5, 4.0, 1.5, 0.0], [1.0, 2, 3, 4, 5, 6], 0))
    # COO rows spread over 300 with 60 present: homes r % 64 collide (ordered insert)
    present = np.sort(rng.choice(300, 60, replace=False))
    rows = np.repeat(present, rng.integers(1, 4, 60))
    cols = np.concatenate([np.sort(rng.choice(40, k, replace=False)) for k in
                           np.bincount(np.searchsorted(present, rows), minlength=60)])
    vals = rng.uniform(-1, 1, len(rows))
    cases.append(hashout_case("ho_coo_collide", 300, 40, rows, cols, vals,
                              rng.uniform(-1, 1, 40), 64))
    # banded 50 x 50, pinned width 53 (odd; all rows inserted, no wrap)
    n = 50
    r = np.repeat(np.arange(n), 3)
    c = np.clip(r + np.tile([-2, 0, 3], n), 0, n - 1)
    key = np.unique(r * n + c)
    cases.append(hashout_case("ho_band_w53", n, n, key // n, key % n, rng.uniform(-1, 1, len(key)),
                              rng.uniform(-1, 1, n), 53))
    return cases


def main():
    out_dir = HERE
    layouts = check_generator_layouts()
    groups = {
        "spmv": lambda: spmv_cases() + [coo_duplicates_case(), dia_case(4, 21), dia_case(5, 22)],
        "add": add_cases,
        "mttkrp": mttkrp_cases,
        "convert": convert_cases,
        "widen": widen_cases,
        "assembly": assembly_cases,
        "io": io_cases,
        "addx": addx_cases,
        "hashout": hashout_cases,
    }
    only = set(sys.argv[1:])
    for group, make in groups.items():
        if only and group not in only:
            continue
        cases = make()
        flat = {}
        names = []
        for name, arrays in cases:
            names.append(name)
            for k, v in arrays.items():
                flat[f"{name}/{k}"] = np.asarray(v)
        flat["_cases"] = np.array(names)
        np.savez_compressed(out_dir / f"{group}.npz", **flat)
        print(group, len(names), "cases")
    if only and "levels" not in only:
        return
    kats = level_kats()
    kats.update(layouts)
    np.savez_compressed(out_dir / "levels.npz", **kats)
    print("levels", len(kats), "tables")


if __name__ == "__main__":
    main()
