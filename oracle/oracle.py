"""numpy wrappers around the C oracle (oracle/sl_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference legs, as the checker or the CPU
baseline.  The product package (paper_1804_10112_b200) never imports it.

Every function follows the reference interpreter's evaluation order (see the
per-function citations in sl_oracle.c) and is pinned against golden vectors
made by running the reference itself (tests/golden/make_golden.py).
Reductions return (out, sum_abs_terms) so callers can apply the
condition-scaled tolerance |gpu - ref| <= 1e-12 * max(|ref|, sum|terms|).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libsl_oracle.so"

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_ptr = ctypes.c_void_p


def build(force: bool = False) -> Path:
    src = HERE / "sl_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        sig = {
            "or_spmv_coo": [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_spmv_coo_mt": [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, ctypes.c_int],
            "or_spmv_csr": [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_spmv_csr_mt": [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, ctypes.c_int],
            "or_spmv_ell": [_i64, _i32, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_spmv_ell_mt": [_i64, _i32, _ptr, _ptr, _ptr, _ptr, ctypes.c_int],
            "or_spmv_dia": [_i64, _i64, _i32, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_spmv_dia_mt": [_i64, _i64, _i32, _ptr, _ptr, _ptr, _ptr, ctypes.c_int],
            "or_hashed_locate": [_i64, _ptr, _ptr, _i64, _ptr, _ptr, _ptr],
            "or_hashed_insert": [_i64, _ptr, _ptr, _i64, _ptr],
            "or_spmv_csr_hashx": [_i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr],
            "or_spmv_csr_hashx_mt": [_i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, ctypes.c_int],
            "or_add_csr": [_i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_add_csr_mt": [_i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                              _ptr, ctypes.c_int],
            "or_mttkrp_coo3": [_i64, _i32, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_mttkrp_coo3_mt": [_i64, _i32, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                                  ctypes.c_int],
            "or_mttkrp_csf": [_i64, _i32, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                              _ptr, _ptr],
            "or_mttkrp_csf_mt": [_i64, _i32, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                                 _ptr, _ptr, ctypes.c_int],
            "or_spmv_csr_spx": [_i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr],
            "or_spmm_csr": [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_spmm_csr_mt": [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, ctypes.c_int],
            "or_ttv_csf": [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_ttm_csf": [_i64, _i32, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_inner_coo3": [_i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr],
            "or_num_threads": [],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
        L.or_add_csr.restype = _i64
        L.or_add_csr_mt.restype = _i64
        L.or_hashed_insert.restype = ctypes.c_int
        L.or_num_threads.restype = ctypes.c_int
        L.or_inner_coo3.restype = ctypes.c_double
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def num_threads() -> int:
    return int(lib().or_num_threads())


def spmv_coo(nrows, rows, cols, vals, x, threads=None):
    rows, cols = _c(rows, np.int32), _c(cols, np.int32)
    vals, x = _c(vals, np.float64), _c(x, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    if threads is None:
        a = np.empty(nrows, dtype=np.float64)
        lib().or_spmv_coo(nrows, len(rows), _p(rows), _p(cols), _p(vals), _p(x), _p(y), _p(a))
        return y, a
    lib().or_spmv_coo_mt(nrows, len(rows), _p(rows), _p(cols), _p(vals), _p(x), _p(y), threads)
    return y


def spmv_csr(nrows, pos, crd, vals, x, threads=None):
    pos, crd = _c(pos, np.int32), _c(crd, np.int32)
    vals, x = _c(vals, np.float64), _c(x, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    if threads is None:
        a = np.empty(nrows, dtype=np.float64)
        lib().or_spmv_csr(nrows, _p(pos), _p(crd), _p(vals), _p(x), _p(y), _p(a))
        return y, a
    lib().or_spmv_csr_mt(nrows, _p(pos), _p(crd), _p(vals), _p(x), _p(y), threads)
    return y


def spmv_ell(nrows, nslots, crd, vals, x, threads=None):
    crd, vals, x = _c(crd, np.int32), _c(vals, np.float64), _c(x, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    if threads is None:
        a = np.empty(nrows, dtype=np.float64)
        lib().or_spmv_ell(nrows, nslots, _p(crd), _p(vals), _p(x), _p(y), _p(a))
        return y, a
    lib().or_spmv_ell_mt(nrows, nslots, _p(crd), _p(vals), _p(x), _p(y), threads)
    return y


def spmv_dia(nrows, ncols, offsets, vals, x, threads=None):
    offsets, vals, x = _c(offsets, np.int32), _c(vals, np.float64), _c(x, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    if threads is None:
        a = np.empty(nrows, dtype=np.float64)
        lib().or_spmv_dia(nrows, ncols, len(offsets), _p(offsets), _p(vals), _p(x), _p(y), _p(a))
        return y, a
    lib().or_spmv_dia_mt(nrows, ncols, len(offsets), _p(offsets), _p(vals), _p(x), _p(y), threads)
    return y


def hashed_locate(coords, w, crd, parent=None):
    coords, crd = _c(coords, np.int32), _c(crd, np.int32)
    parent = _c(parent, np.int32)
    pos = np.empty(len(coords), dtype=np.int32)
    found = np.empty(len(coords), dtype=np.uint8)
    lib().or_hashed_locate(len(coords), _p(parent), _p(coords), w, _p(crd), _p(pos), _p(found))
    return pos, found.astype(bool)


def hashed_insert(coords, w, nseg=1, parent=None, crd=None):
    coords, parent = _c(coords, np.int32), _c(parent, np.int32)
    crd = np.full(nseg * w, -1, dtype=np.int32) if crd is None else _c(crd, np.int32).copy()
    st = lib().or_hashed_insert(len(coords), _p(parent), _p(coords), w, _p(crd))
    return crd, st


def spmv_csr_hashx(nrows, pos, crd, vals, w, xcrd, xvals, threads=None):
    pos, crd, vals = _c(pos, np.int32), _c(crd, np.int32), _c(vals, np.float64)
    xcrd, xvals = _c(xcrd, np.int32), _c(xvals, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    if threads is None:
        a = np.empty(nrows, dtype=np.float64)
        lib().or_spmv_csr_hashx(nrows, _p(pos), _p(crd), _p(vals), w, _p(xcrd), _p(xvals), _p(y),
                                _p(a))
        return y, a
    lib().or_spmv_csr_hashx_mt(nrows, _p(pos), _p(crd), _p(vals), w, _p(xcrd), _p(xvals), _p(y),
                               threads)
    return y


def spmv_csr_spx(nrows, pos, crd, vals, xcrd, xvals):
    """CSR x sparse-vector (intersection), see or_spmv_csr_spx."""
    pos, crd, vals = _c(pos, np.int32), _c(crd, np.int32), _c(vals, np.float64)
    xcrd, xvals = _c(xcrd, np.int32), _c(xvals, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    a = np.empty(nrows, dtype=np.float64)
    lib().or_spmv_csr_spx(nrows, _p(pos), _p(crd), _p(vals), len(xcrd), _p(xcrd), _p(xvals),
                          _p(y), _p(a))
    return y, a


def spmm_csr(nrows, K, pos, crd, vals, X, threads=None):
    """Y = A X with A CSR, X dense (ncols x K), see or_spmm_csr."""
    pos, crd, vals = _c(pos, np.int32), _c(crd, np.int32), _c(vals, np.float64)
    X = _c(X, np.float64)
    Y = np.empty(nrows * K, dtype=np.float64)
    if threads is None:
        a = np.empty(nrows * K, dtype=np.float64)
        lib().or_spmm_csr(nrows, K, _p(pos), _p(crd), _p(vals), _p(X), _p(Y), _p(a))
        return Y.reshape(nrows, K), a.reshape(nrows, K)
    lib().or_spmm_csr_mt(nrows, K, _p(pos), _p(crd), _p(vals), _p(X), _p(Y), threads)
    return Y.reshape(nrows, K)


def ttv_csf(csf, vals, v):
    """Fiber sums of TTV over a CSF tensor (dict with pos0..crd2): (sums, abs sums)."""
    c = {k: _c(csf[k], np.int32) for k in ("crd0", "pos1", "crd1", "pos2", "crd2")}
    vals, v = _c(vals, np.float64), _c(v, np.float64)
    nf = len(c["crd1"])
    out, a = np.empty(nf, np.float64), np.empty(nf, np.float64)
    lib().or_ttv_csf(len(c["crd0"]), _p(c["crd0"]), _p(c["pos1"]), _p(c["crd1"]), _p(c["pos2"]),
                     _p(c["crd2"]), _p(vals), _p(v), _p(out), _p(a))
    return out, a


def ttm_csf(csf, vals, U):
    """One R-row per fiber of TTM over a CSF tensor (nfibers x R)."""
    c = {k: _c(csf[k], np.int32) for k in ("crd0", "pos1", "pos2", "crd2")}
    vals, U = _c(vals, np.float64), _c(U, np.float64)
    R = U.shape[1]
    out = np.empty((len(_c(csf["crd1"], np.int32)), R), np.float64)
    lib().or_ttm_csf(len(c["crd0"]), R, _p(c["pos1"]), _p(c["pos2"]), _p(c["crd2"]), _p(vals),
                     _p(U), _p(out))
    return out


def inner_coo3(x, z):
    """a() = X(i,j,k) * Z(i,j,k) over two sorted COO-3 tensors (dicts i, j, k, vals)."""
    xs = [_c(x[k], np.int32) for k in ("i", "j", "k")] + [_c(x["vals"], np.float64)]
    zs = [_c(z[k], np.int32) for k in ("i", "j", "k")] + [_c(z["vals"], np.float64)]
    a = np.zeros(1, np.float64)
    r = lib().or_inner_coo3(len(xs[0]), *[_p(t) for t in xs], len(zs[0]),
                            *[_p(t) for t in zs], _p(a))
    return float(r), float(a[0])


def add_csr(nrows, a_pos, a_crd, a_vals, b_cols, b_vals, b_rows=None, b_pos=None, threads=None):
    a_pos, a_crd, a_vals = _c(a_pos, np.int32), _c(a_crd, np.int32), _c(a_vals, np.float64)
    b_cols, b_vals = _c(b_cols, np.int32), _c(b_vals, np.float64)
    b_rows, b_pos = _c(b_rows, np.int32), _c(b_pos, np.int32)
    cap = len(a_crd) + len(b_cols)
    c_pos = np.empty(nrows + 1, dtype=np.int32)
    c_crd = np.empty(max(cap, 1), dtype=np.int32)
    c_vals = np.empty(max(cap, 1), dtype=np.float64)
    args = (nrows, _p(a_pos), _p(a_crd), _p(a_vals), len(b_cols), _p(b_pos), _p(b_rows),
            _p(b_cols), _p(b_vals), _p(c_pos), _p(c_crd), _p(c_vals))
    if threads is None:
        n = lib().or_add_csr(*args)
    else:
        n = lib().or_add_csr_mt(*args, threads)
    return c_pos, c_crd[:n].copy(), c_vals[:n].copy()


def mttkrp_coo3(I, i, j, k, vals, B, C, threads=None):
    i, j, k = _c(i, np.int32), _c(j, np.int32), _c(k, np.int32)
    vals, B, C = _c(vals, np.float64), _c(B, np.float64), _c(C, np.float64)
    R = B.shape[1]
    A = np.empty((I, R), dtype=np.float64)
    if threads is None:
        a = np.empty((I, R), dtype=np.float64)
        lib().or_mttkrp_coo3(I, R, len(i), _p(i), _p(j), _p(k), _p(vals), _p(B), _p(C), _p(A),
                             _p(a))
        return A, a
    lib().or_mttkrp_coo3_mt(I, R, len(i), _p(i), _p(j), _p(k), _p(vals), _p(B), _p(C), _p(A),
                            threads)
    return A


def mttkrp_csf(I, crd0, pos1, crd1, pos2, crd2, vals, B, C, threads=None):
    crd0, pos1, crd1 = _c(crd0, np.int32), _c(pos1, np.int32), _c(crd1, np.int32)
    pos2, crd2 = _c(pos2, np.int32), _c(crd2, np.int32)
    vals, B, C = _c(vals, np.float64), _c(B, np.float64), _c(C, np.float64)
    R = B.shape[1]
    A = np.empty((I, R), dtype=np.float64)
    if threads is None:
        a = np.empty((I, R), dtype=np.float64)
        lib().or_mttkrp_csf(I, R, len(crd0), _p(crd0), _p(pos1), _p(crd1), _p(pos2), _p(crd2),
                            _p(vals), _p(B), _p(C), _p(A), _p(a))
        return A, a
    lib().or_mttkrp_csf_mt(I, R, len(crd0), _p(crd0), _p(pos1), _p(crd1), _p(pos2), _p(crd2),
                           _p(vals), _p(B), _p(C), _p(A), threads)
    return A


# ---- format conversion (formats.convert -> engine.identity_copy,
#      formats.py:583-587, engine.py:775-779) -------------------------------

def convert_coo_to_csr(nrows, rows, cols, vals, threads=None):
    """Identity copy COO -> CSR = gather-append writer over the COO's grouped
    rows/columns (engine.py:330-434): the A+B restatement with A empty."""
    a_pos = np.zeros(nrows + 1, dtype=np.int32)
    e_i = np.zeros(0, dtype=np.int32)
    e_f = np.zeros(0, dtype=np.float64)
    return add_csr(nrows, a_pos, e_i, e_f, cols, vals, b_rows=rows, threads=threads)


def convert_csr_to_ell(nrows, pos, crd, vals):
    """Identity copy -> ELL goes through the reorder writer (cells[key] =
    0.0 + v, engine.py:437-452) and assemble, whose canonicalize drops exact
    zeros (formats.py:217-222); ELL layout slot-major s*N + i with padding
    (col 0, 0.0), nslots = longest row (formats.py:322-335, 443-455)."""
    pos = np.asarray(pos, dtype=np.int64)
    crd = np.asarray(crd, dtype=np.int32)
    vals = np.asarray(vals, dtype=np.float64)
    keep = vals != 0.0
    row = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(pos))[keep]
    kc, kv = crd[keep], 0.0 + vals[keep]
    counts = np.bincount(row, minlength=nrows) if nrows else np.zeros(0, np.int64)
    nslots = int(counts.max()) if len(kc) else 0
    start = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    slot = np.arange(len(kc), dtype=np.int64) - start[row]
    ecrd = np.zeros(nslots * nrows, dtype=np.int32)
    evals = np.zeros(nslots * nrows, dtype=np.float64)
    ecrd[slot * nrows + row] = kc
    evals[slot * nrows + row] = kv
    return nslots, ecrd, evals


def convert_coo_to_dia(nrows, ncols, rows, cols, vals):
    """Identity copy -> DIA (unique coordinates): reorder writer + assemble;
    offsets = sorted distinct c - r of the kept entries (formats.py:313),
    vals[d*N + r] (formats.py:405-412), 0.0 elsewhere."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    keep = vals != 0.0
    r, c, v = rows[keep], cols[keep], 0.0 + vals[keep]
    offs = np.unique(c - r).astype(np.int32)
    d = np.searchsorted(offs, c - r)
    dvals = np.zeros(len(offs) * nrows, dtype=np.float64)
    dvals[d * nrows + r] = v
    return offs, dvals


def bits_equal(a, b) -> bool:
    """Bit-exact equality of float64 arrays, treating +0.0 and -0.0 as different."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and bool(np.array_equal(a.view(np.int64), b.view(np.int64)))


def within_condition(gpu, ref, sum_abs, rtol=1e-12):
    """Condition-scaled check |gpu - ref| <= rtol * max(|ref|, sum|terms|)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.maximum(np.abs(ref), np.asarray(sum_abs, dtype=np.float64))
    err = np.abs(gpu - ref)
    ok = err <= rtol * scale
    return bool(ok.all()), float((err / np.where(scale > 0, scale, 1.0)).max(initial=0.0))


if os.environ.get("SL_ORACLE_BUILD") == "1":  # pragma: no cover
    build(force=True)
