"""Thin tensor-level wrappers over the C ABI (include/sl_abi.h).

Each function takes CUDA tensors in the reference's storage layouts, checks
dtype/device/contiguity, allocates outputs and workspace with the torch
caching allocator, and launches on the current stream.  Nothing here runs on
the CPU: a non-CUDA tensor raises DeviceError.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DeviceError

I32, F64 = torch.int32, torch.float64


def _t(x, dtype, name):
    if not isinstance(x, torch.Tensor):
        raise DeviceError(f"{name} must be a CUDA tensor, got {type(x).__name__}")
    if not x.is_cuda:
        raise DeviceError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if x.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {x.dtype}")
    return x if x.is_contiguous() else x.contiguous()


def _out(y, n, dtype, like, name):
    if y is None:
        return torch.empty(n, dtype=dtype, device=like.device)
    y = _t(y, dtype, name)
    if y.numel() < n:
        raise ValueError(f"{name} has {y.numel()} elements, needs {n}")
    return y


def _ws(nbytes, like):
    if nbytes == 0:
        return None
    return torch.empty(int(nbytes), dtype=torch.uint8, device=like.device)


L = _lib.load
S = _lib.stream_handle
P = _lib.ptr


# ---- SpMV -------------------------------------------------------------------

def spmv_coo(nrows, ncols, rows, cols, vals, x, y=None, ws=None, direct=False):
    """COO SpMV.  The workspace holds the row level's position index, built
    per call; direct=True runs the staged-tile kernel on the coordinates
    alone (no workspace)."""
    rows, cols = _t(rows, I32, "rows"), _t(cols, I32, "cols")
    vals, x = _t(vals, F64, "vals"), _t(x, F64, "x")
    y = _out(y, nrows, F64, x, "y")
    if direct:
        ws = None
    elif ws is None:
        ws = _ws(L().sl_spmv_coo_workspace_bytes(nrows), x)
    _lib.check(L().sl_spmv_coo_f64(nrows, ncols, rows.numel(), P(rows), P(cols), P(vals), P(x),
                                   P(y), P(ws), 0 if ws is None else ws.numel(), S()), "spmv_coo")
    return y


def spmv_csr(nrows, ncols, pos, crd, vals, x, y=None, variant=0, ws=None):
    pos, crd = _t(pos, I32, "pos"), _t(crd, I32, "crd")
    vals, x = _t(vals, F64, "vals"), _t(x, F64, "x")
    y = _out(y, nrows, F64, x, "y")
    nnz = crd.numel()
    lib = L()
    if variant == 2:                     # only the merge-path split uses a workspace
        need = lib.sl_spmv_csr_workspace_bytes(nrows, nnz, variant)
        if ws is None or ws.numel() < need:
            ws = _ws(need, x)
    st = lib.sl_spmv_csr_f64(nrows, ncols, nnz, pos.data_ptr(), crd.data_ptr(), vals.data_ptr(),
                             x.data_ptr(), y.data_ptr(), variant, P(ws),
                             0 if ws is None else ws.numel(), S())
    if st:
        _lib.check(st, "spmv_csr")
    return y


def spmv_csr_peers(nrows, ncols, pos, crd, vals, x, peer_ptrs):
    """CSR SpMV of a row block storing every row into each buffer of
    `peer_ptrs` (device pointers, already offset to the block's first row):
    the all-gather of y fused into the kernel's epilogue (sl_spmv_csr_peers_f64)."""
    import ctypes

    pos, crd = _t(pos, I32, "pos"), _t(crd, I32, "crd")
    vals, x = _t(vals, F64, "vals"), _t(x, F64, "x")
    arr = (ctypes.c_uint64 * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
    _lib.check(L().sl_spmv_csr_peers_f64(nrows, ncols, crd.numel(), P(pos), P(crd), P(vals), P(x),
                                         ctypes.cast(arr, ctypes.c_void_p), len(peer_ptrs), S()),
               "spmv_csr_peers")


def spmv_ell(nrows, ncols, nslots, crd, vals, x, y=None):
    crd, vals, x = _t(crd, I32, "crd"), _t(vals, F64, "vals"), _t(x, F64, "x")
    y = _out(y, nrows, F64, x, "y")
    _lib.check(L().sl_spmv_ell_f64(nrows, ncols, nslots, P(crd), P(vals), P(x), P(y), S()),
               "spmv_ell")
    return y


def spmv_dia(nrows, ncols, offsets, vals, x, y=None, row0=0):
    """`offsets`: host numpy int32 (passed as kernel parameters) or a CUDA
    tensor.  row0 > 0 evaluates the row block [row0, row0 + nrows) of a larger
    matrix (vals hold the block's slots, x the whole vector)."""
    vals, x = _t(vals, F64, "vals"), _t(x, F64, "x")
    y = _out(y, nrows, F64, x, "y")
    if isinstance(offsets, torch.Tensor) and offsets.is_cuda:
        offs = _t(offsets, I32, "offsets")
        nd, optr, on_host = offs.numel(), P(offs), 0
    else:
        offs = np.ascontiguousarray(offsets, dtype=np.int32)
        nd, optr, on_host = len(offs), offs.ctypes.data, 1
        if nd > 32:
            return spmv_dia(nrows, ncols, torch.as_tensor(offs, device=x.device), vals, x, y, row0)
    _lib.check(L().sl_spmv_dia_rows_f64(nrows, row0, ncols, nd, optr, on_host, P(vals), P(x),
                                        P(y), S()), "spmv_dia")
    return y


def spmv_csr_hashx(nrows, pos, crd, vals, w, x_crd, x_vals, y=None, n=None, ws=None):
    """CSR x hash-vector.  With the vector's dimension `n`, the slot-map path
    (sl_spmv_csr_hashx_map_f64: one locate per coordinate) runs; without it,
    every nonzero probes the table (sl_spmv_csr_hashx_f64).  Same results."""
    pos, crd, vals = _t(pos, I32, "pos"), _t(crd, I32, "crd"), _t(vals, F64, "vals")
    x_crd, x_vals = _t(x_crd, I32, "x_crd"), _t(x_vals, F64, "x_vals")
    y = _out(y, nrows, F64, vals, "y")
    if n is None:
        _lib.check(L().sl_spmv_csr_hashx_f64(nrows, P(pos), P(crd), P(vals), w, P(x_crd),
                                             P(x_vals), P(y), S()), "spmv_csr_hashx")
        return y
    need = L().sl_spmv_csr_hashx_map_workspace_bytes(n, w)
    if ws is None or ws.numel() < need:
        ws = _ws(need, vals)
    _lib.check(L().sl_spmv_csr_hashx_map_f64(nrows, n, crd.numel(), P(pos), P(crd), P(vals), w,
                                             P(x_crd),
                                             P(x_vals), P(y), P(ws), ws.numel(), S()),
               "spmv_csr_hashx_map")
    return y


def spmv_csr_spx(nrows, n, pos, crd, vals, x_crd, x_vals, y=None, ws=None):
    """CSR x sparse-vector (intersection), x of dimension n."""
    pos, crd, vals = _t(pos, I32, "pos"), _t(crd, I32, "crd"), _t(vals, F64, "vals")
    x_crd, x_vals = _t(x_crd, I32, "x_crd"), _t(x_vals, F64, "x_vals")
    y = _out(y, nrows, F64, vals, "y")
    need = L().sl_spmv_csr_spx_workspace_bytes(n)
    if ws is None or ws.numel() < need:
        ws = _ws(need, vals)
    _lib.check(L().sl_spmv_csr_spx_f64(nrows, n, crd.numel(), P(pos), P(crd), P(vals),
                                       x_crd.numel(), P(x_crd),
                                       P(x_vals), P(y), P(ws), ws.numel(), S()), "spmv_csr_spx")
    return y


def spmm_csr(nrows, ncols, pos, crd, vals, X, Y=None, long_min=None):
    """Y = A X, A CSR (nrows x ncols), X dense (ncols x K) row-major.  With
    `long_min`, rows longer than it run one CTA per row
    (sl_spmm_csr_split_f64); same results."""
    pos, crd, vals = _t(pos, I32, "pos"), _t(crd, I32, "crd"), _t(vals, F64, "vals")
    X = _t(X, F64, "X")
    K = X.shape[-1] if X.dim() == 2 else X.numel() // max(ncols, 1)
    Y = _out(Y, nrows * K, F64, vals, "Y").view(nrows, K) if Y is None else _t(Y, F64, "Y")
    nnz = crd.numel()
    if long_min is None:
        _lib.check(L().sl_spmm_csr_nnz_f64(nrows, ncols, K, nnz, P(pos), P(crd), P(vals), P(X),
                                           P(Y), S()), "spmm_csr")
        return Y
    ws = _ws(L().sl_spmm_csr_split_workspace_bytes(nrows, nnz, long_min), vals)
    _lib.check(L().sl_spmm_csr_split_f64(nrows, ncols, K, nnz, P(pos), P(crd), P(vals), P(X),
                                         P(Y), long_min, P(ws), 0 if ws is None else ws.numel(),
                                         S()), "spmm_csr")
    return Y


# ---- 3-tensor kernels beyond MTTKRP ---------------------------------------------

def _fibers(crd0, pos1, crd1, pos2, crd2, vals):
    return (_t(crd0, I32, "crd0"), _t(pos1, I32, "pos1"), _t(crd1, I32, "crd1"),
            _t(pos2, I32, "pos2"), _t(crd2, I32, "crd2"), _t(vals, F64, "vals"))


def ttv_csf(I, J, K, crd0, pos1, crd1, pos2, crd2, vals, v, out="dense"):
    """TTV over a CSF tensor.  out="dense": (I, J) tensor; out="csr":
    (pos, crd, vals) with one entry per fiber."""
    crd0, pos1, crd1, pos2, crd2, vals = _fibers(crd0, pos1, crd1, pos2, crd2, vals)
    v = _t(v, F64, "v")
    nf = crd1.numel()
    sums = torch.empty(nf, dtype=F64, device=vals.device)
    if nf:
        # fibre lengths are typically power-law (Zipf slices): the merge-path
        # split keeps a few huge fibres from serialising one warp (D5: 0.23 ms
        # against 2.6 ms with the register hand-off, 7.5 ms with the row-block)
        spmv_csr(nf, K, pos2, crd2, vals, v, sums, variant=2)
    if out == "csr":
        pos = torch.empty(I + 1, dtype=I32, device=vals.device)
        _lib.check(L().sl_csf_fiber_rowptr(I, crd0.numel(), P(crd0), P(pos1), P(pos), S()),
                   "csf_fiber_rowptr")
        return pos, crd1.clone(), sums
    Y = torch.empty((I, J), dtype=F64, device=vals.device)
    _lib.check(L().sl_csf_fiber_scatter_f64(I, J, 1, crd0.numel(), nf, P(crd0), P(pos1), P(crd1),
                                            P(sums), P(Y), S()), "csf_fiber_scatter")
    return Y


def ttm_csf(I, J, K, crd0, pos1, crd1, pos2, crd2, vals, U, long_min=None):
    """TTM over a CSF tensor: Y (I, J, R) dense.  `long_min`: fibres longer
    than it take the SpMM long-row split (same results)."""
    crd0, pos1, crd1, pos2, crd2, vals = _fibers(crd0, pos1, crd1, pos2, crd2, vals)
    U = _t(U, F64, "U")
    R = U.shape[-1]
    nf = crd1.numel()
    rows = torch.empty((nf, R), dtype=F64, device=vals.device)
    if nf:
        spmm_csr(nf, K, pos2, crd2, vals, U.view(K, R), rows, long_min=long_min)
    Y = torch.empty((I, J, R), dtype=F64, device=vals.device)
    _lib.check(L().sl_csf_fiber_scatter_f64(I, J, R, crd0.numel(), nf, P(crd0), P(pos1), P(crd1),
                                            P(rows), P(Y), S()), "csf_fiber_scatter")
    return Y


def inner_coo3(I, J, K, x, z):
    """a() = X(i,j,k) * Z(i,j,k) over two sorted COO-3 tensors given as
    (i, j, k, vals) tuples of CUDA tensors; returns a 1-element device tensor."""
    xi, xj, xk, xv = (_t(t, d, n) for t, d, n in zip(x, (I32, I32, I32, F64), "ijkv"))
    zi, zj, zk, zv = (_t(t, d, n) for t, d, n in zip(z, (I32, I32, I32, F64), "ijkv"))
    out = torch.empty(1, dtype=F64, device=xv.device)
    ws = _ws(L().sl_inner_coo3_workspace_bytes(xi.numel()), xv)
    _lib.check(L().sl_inner_coo3_f64(I, J, K, xi.numel(), P(xi), P(xj), P(xk), P(xv), zi.numel(),
                                     P(zi), P(zj), P(zk), P(zv), P(out), P(ws), ws.numel(), S()),
               "inner_coo3")
    return out


def hashed_slot_map(n, w, crd, ws=None):
    """u64 per coordinate c < n: (probe distance << 32 | slot) of locate(c), ~0 absent."""
    crd = _t(crd, I32, "crd")
    need = L().sl_hashed_slot_map_workspace_bytes(n, w)
    if ws is None or ws.numel() < need:
        ws = _ws(need, crd)
    _lib.check(L().sl_hashed_slot_map(n, w, P(crd), P(ws), ws.numel(), S()), "hashed_slot_map")
    return ws[:8 * n].view(torch.int64)


# ---- hashed level -------------------------------------------------------------

def hashed_locate(coords, w, crd, parent=None, group=8):
    coords, crd = _t(coords, I32, "coords"), _t(crd, I32, "crd")
    parent = None if parent is None else _t(parent, I32, "parent")
    pos = torch.empty(coords.numel(), dtype=I32, device=coords.device)
    found = torch.empty(coords.numel(), dtype=torch.uint8, device=coords.device)
    _lib.check(L().sl_hashed_locate(coords.numel(), P(parent), P(coords), w, P(crd), P(pos),
                                    P(found), group, S()), "hashed_locate")
    return pos, found


def hashed_insert(coords, w, nseg=1, parent=None, crd=None, ordered=True):
    """Bulk hashed insert; returns (crd table, device error flag).  ordered:
    the exact table the sequential insert_coord calls build (default);
    ordered=False: the concurrent atomicCAS insert (same stored set per
    segment, layout unspecified where probe sequences collide)."""
    coords = _t(coords, I32, "coords")
    parent = None if parent is None else _t(parent, I32, "parent")
    if crd is None:
        crd = torch.empty(nseg * w, dtype=I32, device=coords.device)
        _lib.check(L().sl_hashed_insert_init(crd.numel(), P(crd), S()), "insert_init")
    err = torch.zeros(1, dtype=I32, device=coords.device)
    if ordered:
        ws = _ws(L().sl_hashed_insert_ordered_workspace_bytes(coords.numel(), crd.numel()), crd)
        _lib.check(L().sl_hashed_insert_ordered(coords.numel(), P(parent), P(coords), w,
                                                crd.numel(), P(crd), P(err), P(ws),
                                                0 if ws is None else ws.numel(), S()),
                   "hashed_insert")
    else:
        _lib.check(L().sl_hashed_insert(coords.numel(), P(parent), P(coords), w, P(crd), P(err),
                                        S()), "hashed_insert")
    return crd, err


# ---- C = A + B -----------------------------------------------------------------

def add_csr(nrows, a_pos, a_crd, a_vals, b_cols, b_vals, b_rows=None, b_pos=None, sync=True,
            two_pass=False):
    """CSR + (COO | CSR) -> CSR.  Returns (c_pos, c_crd, c_vals); with
    sync=False the crd/vals buffers are upper-bound sized (nnz_a + nnz_b) and
    nnz_c = c_pos[nrows] is left on the device.  two_pass=True runs the
    count -> scan -> fill pair (sl_add_csr_count / sl_add_csr_fill), the
    default the fused single pass (sl_add_csr_f64); both are bit-identical."""
    a_pos, a_crd, a_vals = _t(a_pos, I32, "a_pos"), _t(a_crd, I32, "a_crd"), _t(a_vals, F64, "a_vals")
    b_cols, b_vals = _t(b_cols, I32, "b_cols"), _t(b_vals, F64, "b_vals")
    b_rows = None if b_rows is None else _t(b_rows, I32, "b_rows")
    b_pos = None if b_pos is None else _t(b_pos, I32, "b_pos")
    bnnz = b_cols.numel()
    dev = a_vals.device
    c_pos = torch.empty(nrows + 1, dtype=I32, device=dev)
    cap = max(a_crd.numel() + bnnz, 1)
    c_crd = torch.empty(cap, dtype=I32, device=dev)
    c_vals = torch.empty(cap, dtype=F64, device=dev)
    need = L().sl_add_csr_workspace_bytes(nrows, bnnz)
    ws = _ws(need, a_vals)
    wsn = 0 if ws is None else ws.numel()
    if two_pass:
        _lib.check(L().sl_add_csr_count(nrows, P(a_pos), P(a_crd), bnnz, P(b_pos), P(b_rows),
                                        P(b_cols), P(c_pos), P(ws), wsn, S()), "add_count")
        _lib.check(L().sl_add_csr_fill(nrows, P(a_pos), P(a_crd), P(a_vals), bnnz, P(b_pos),
                                       P(b_rows), P(b_cols), P(b_vals), P(c_pos), P(c_crd),
                                       P(c_vals), P(ws), wsn, S()), "add_fill")
    else:
        _lib.check(L().sl_add_csr_f64(nrows, P(a_pos), P(a_crd), P(a_vals), bnnz, P(b_pos),
                                      P(b_rows), P(b_cols), P(b_vals), P(c_pos), P(c_crd),
                                      P(c_vals), P(ws), wsn, S()), "add_csr")
    if sync:
        n = int(c_pos[nrows].item())
        return c_pos, c_crd[:n], c_vals[:n]
    return c_pos, c_crd, c_vals


# ---- format conversion (formats.convert, formats.py:583-587) -------------------

def coo_to_csr(nrows, rows, cols, vals, sync=True, two_pass=True, path="exact"):
    """COO-SoA -> CSR exactly as the reference's identity copy: duplicates
    summed (+0.0 + v1 + v2 ...), values stored as 0.0 + v (explicit zeros
    kept).  Default: sl_convert_coo_to_csr_exact (one streaming pass when no
    coordinate repeats, the A+B gather-append passes otherwise, decided on the
    device).  path="add" routes through the A+B entry points with an empty A
    (two_pass selecting the two-pass or fused form, as add_csr), for A/B
    checks."""
    rows = _t(rows, I32, "rows")
    if path == "add":
        a_pos = torch.zeros(nrows + 1, dtype=I32, device=rows.device)
        empty_i = torch.empty(0, dtype=I32, device=rows.device)
        empty_f = torch.empty(0, dtype=F64, device=rows.device)
        return add_csr(nrows, a_pos, empty_i, empty_f, cols, vals, b_rows=rows, sync=sync,
                       two_pass=two_pass)
    cols, vals = _t(cols, I32, "cols"), _t(vals, F64, "vals")
    nnz = rows.numel()
    dev = rows.device
    c_pos = torch.empty(nrows + 1, dtype=I32, device=dev)
    c_crd = torch.empty(max(nnz, 1), dtype=I32, device=dev)
    c_vals = torch.empty(max(nnz, 1), dtype=F64, device=dev)
    ws = _ws(L().sl_convert_coo_to_csr_exact_workspace_bytes(nrows, nnz), vals)
    _lib.check(L().sl_convert_coo_to_csr_exact(nrows, nnz, P(rows), P(cols), P(vals), P(c_pos),
                                               P(c_crd), P(c_vals), P(ws),
                                               0 if ws is None else ws.numel(), S()),
               "convert_coo_to_csr")
    if sync:
        n = int(c_pos[nrows].item())
        return c_pos, c_crd[:n], c_vals[:n]
    return c_pos, c_crd, c_vals


def csr_rows(nrows, pos, nnz=None):
    """COO row coordinates of a CSR structure."""
    pos = _t(pos, I32, "pos")
    nnz = int(pos[nrows].item()) if nnz is None else nnz
    rows = torch.empty(nnz, dtype=I32, device=pos.device)
    _lib.check(L().sl_csr_row_indices(nrows, P(pos), P(rows), S()), "csr_rows")
    return rows


def csr_to_coo(nrows, pos, crd, vals):
    """CSR -> COO-SoA exactly as the identity copy: gather-append of 0.0 + v
    (the A+B kernels with an empty B), explicit zeros kept."""
    pos, crd, vals = _t(pos, I32, "pos"), _t(crd, I32, "crd"), _t(vals, F64, "vals")
    e_i = torch.empty(0, dtype=I32, device=pos.device)
    e_f = torch.empty(0, dtype=F64, device=pos.device)
    b_pos = torch.zeros(nrows + 1, dtype=I32, device=pos.device)
    c_pos, c_crd, c_vals = add_csr(nrows, pos, crd, vals, e_i, e_f, b_pos=b_pos)
    return csr_rows(nrows, c_pos, c_crd.numel()), c_crd, c_vals


def coo_rowptr(nrows, rows, pos=None):
    """Structural part alone: the row pointer of a row-sorted COO."""
    rows = _t(rows, I32, "rows")
    pos = _out(pos, nrows + 1, I32, rows, "pos")
    _lib.check(L().sl_convert_coo_to_csr(nrows, rows.numel(), P(rows), P(pos), S()), "coo_rowptr")
    return pos


def csr_to_ell(nrows, pos, crd, vals):
    """CSR -> ELL (slot-major, padding (0, 0.0)); zeros dropped as assemble
    does.  Returns (nslots, crd, vals); reads nslots back (one sync)."""
    pos, crd, vals = _t(pos, I32, "pos"), _t(crd, I32, "crd"), _t(vals, F64, "vals")
    m = torch.empty(1, dtype=I32, device=pos.device)
    _lib.check(L().sl_csr_max_row_length(nrows, P(pos), P(vals), P(m), S()), "csr_max_row")
    nslots = int(m.item())
    ecrd = torch.empty(nslots * nrows, dtype=I32, device=pos.device)
    evals = torch.empty(nslots * nrows, dtype=F64, device=pos.device)
    _lib.check(L().sl_convert_csr_to_ell(nrows, nslots, P(pos), P(crd), P(vals), P(ecrd),
                                         P(evals), S()), "csr_to_ell")
    return nslots, ecrd, evals


def coo_to_dia(nrows, ncols, rows, cols, vals):
    """COO (unique coordinates) -> DIA.  Returns (offsets, vals); reads the
    diagonal count back (one sync)."""
    rows, cols, vals = _t(rows, I32, "rows"), _t(cols, I32, "cols"), _t(vals, F64, "vals")
    dev = rows.device
    ws = _ws(L().sl_convert_coo_to_dia_workspace_bytes(nrows, ncols), rows)
    offs = torch.empty(nrows + ncols - 1, dtype=I32, device=dev)
    nd = torch.empty(1, dtype=I32, device=dev)
    nnz = rows.numel()
    _lib.check(L().sl_convert_coo_to_dia_offsets(nrows, ncols, nnz, P(rows), P(cols), P(vals),
                                                 P(offs), P(nd), P(ws), ws.numel(), S()),
               "coo_to_dia_offsets")
    ndiag = int(nd.item())
    dvals = torch.empty(ndiag * nrows, dtype=F64, device=dev)
    _lib.check(L().sl_convert_coo_to_dia_values(nrows, ncols, nnz, ndiag, P(rows), P(cols),
                                                P(vals), P(dvals), P(ws), ws.numel(), S()),
               "coo_to_dia_values")
    return offs[:ndiag].clone(), dvals


# ---- MTTKRP ---------------------------------------------------------------------

def _mttkrp_ws(nnz, R, like, ws):
    need = L().sl_mttkrp_workspace_bytes(nnz, R)
    if ws is not None and ws.numel() >= need:
        return ws
    return _ws(need, like)


_MT_MAX_R = 128   # ranks per launch (sl_mttkrp_*: SL_ERR_RANGE above)


def _mttkrp_rank_blocks(fn, I, B, C, A):
    """A(i, r) depends on column r of B and C alone, so ranks beyond one
    launch's limit are computed in column blocks (identical results)."""
    R = B.shape[-1]
    A = torch.empty((I, R), dtype=F64, device=B.device) if A is None else A
    for r0 in range(0, R, _MT_MAX_R):
        r1 = min(R, r0 + _MT_MAX_R)
        A[:, r0:r1] = fn(B[:, r0:r1].contiguous(), C[:, r0:r1].contiguous())
    return A


def mttkrp_coo3(I, J, K, i, j, k, vals, B, C, A=None, ws=None):
    i, j, k = _t(i, I32, "i"), _t(j, I32, "j"), _t(k, I32, "k")
    vals, B, C = _t(vals, F64, "vals"), _t(B, F64, "B"), _t(C, F64, "C")
    R = B.shape[-1]
    if R > _MT_MAX_R:
        return _mttkrp_rank_blocks(lambda b, c: mttkrp_coo3(I, J, K, i, j, k, vals, b, c),
                                   I, B, C, A)
    A = _out(A, I * R, F64, vals, "A").view(I, R) if A is None else _t(A, F64, "A")
    ws = _mttkrp_ws(i.numel(), R, vals, ws)
    _lib.check(L().sl_mttkrp_coo3_f64(I, J, K, R, i.numel(), P(i), P(j), P(k), P(vals), P(B),
                                      P(C), P(A), P(ws), 0 if ws is None else ws.numel(), S()),
               "mttkrp_coo3")
    return A


def mttkrp_csf(I, J, K, crd0, pos1, crd1, pos2, crd2, vals, B, C, A=None, ws=None):
    crd0, pos1, crd1 = _t(crd0, I32, "crd0"), _t(pos1, I32, "pos1"), _t(crd1, I32, "crd1")
    pos2, crd2 = _t(pos2, I32, "pos2"), _t(crd2, I32, "crd2")
    vals, B, C = _t(vals, F64, "vals"), _t(B, F64, "B"), _t(C, F64, "C")
    R = B.shape[-1]
    if R > _MT_MAX_R:
        return _mttkrp_rank_blocks(
            lambda b, c: mttkrp_csf(I, J, K, crd0, pos1, crd1, pos2, crd2, vals, b, c), I, B, C, A)
    A = _out(A, I * R, F64, vals, "A").view(I, R) if A is None else _t(A, F64, "A")
    ws = _mttkrp_ws(vals.numel(), R, vals, ws)
    _lib.check(L().sl_mttkrp_csf_f64(I, J, K, R, crd0.numel(), crd1.numel(), vals.numel(),
                                     P(crd0), P(pos1), P(crd1), P(pos2), P(crd2), P(vals), P(B),
                                     P(C), P(A), P(ws), 0 if ws is None else ws.numel(), S()),
               "mttkrp_csf")
    return A


def l2_flush(buf):
    buf = _t(buf, torch.uint8, "buf")
    _lib.check(L().sl_l2_flush(P(buf), buf.numel(), S()), "l2_flush")


def l2_read(buf, sink):
    buf = _t(buf, torch.uint8, "buf")
    _lib.check(L().sl_l2_read(P(buf), buf.numel(), P(sink), S()), "l2_read")
