"""`evaluate` — the reference's entry point (engine.py:739-764), B200 backend.

The reference plans every expression into a merge-lattice schedule and
interprets it (engine.py:580-713).  For the hot path, the schedules of the
five BASELINE patterns are fixed; `plan` recognises an
(expression, level-kinds) pair as one of them and binds it to the sm_100a
kernel that executes that schedule with the level functions inlined:

    y(i) = A(i,j) * x(j)   A coo-soa | csr | ell | dia, x dense   -> K1..K4
                           A csr, x hash-vector                   -> K5 (locate)
    C(i,j) = A(i,j) + B(i,j)   A csr, B coo-soa | csr, C csr      -> K6
    A(i,r) = X(i,j,k) * B(j,r) * C(k,r)   X coo-3 | csf, B/C dense -> K7 / K8

Anything else raises UnsupportedMergeError (no kernel for that merge) or
UnsupportedOutputError (output format the kernel cannot produce) — there is
no interpreter fallback and no CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence, Tuple

import numpy as np
import torch

from . import kernels as K
from .errors import (HashSegmentFullError, UnsupportedMergeError, UnsupportedOutputError,
                     ValidationError)
from .formats import TensorFormat, TensorStorage, preset
from .levels import LevelKind as LK
from .levels import LevelStorage
from .notation import Access, Add, Assignment, CheckedExpr, Mul, parse, validate


@dataclass
class EvalStats:
    """Visit counters keyed by loop variable and by (variable, lattice-point
    label) (engine.py:255-268).  The GPU path fills them with the visit
    counts the reference's schedule performs — from the storage sizes, and
    for merged streams (A + B unions, intersections) from the coordinates on
    the device — so `by_loop` compares entry for entry with the reference's
    (tests/test_gpu_sweep.py)."""

    by_var: Dict[str, int] = field(default_factory=dict)
    by_loop: Dict[Tuple[str, str], int] = field(default_factory=dict)

    def count(self, var: str, point_label: str, n: int = 1) -> None:
        self.by_var[var] = self.by_var.get(var, 0) + n
        key = (var, point_label)
        self.by_loop[key] = self.by_loop.get(key, 0) + n

    def total(self) -> int:
        return sum(self.by_var.values())


# ---------------------------------------------------------------------------
# format recognition (by level kinds and roles, not by name)

def _whole(fmt: TensorFormat) -> bool:
    return all(r.part == "whole" for r in fmt.roles) and fmt.mode_ordering == tuple(
        range(fmt.order)) and not fmt.aos


def format_class(fmt: TensorFormat) -> str:
    k = fmt.kinds()
    if _whole(fmt):
        if all(x is LK.DENSE for x in k):
            return f"dense{len(k)}"
        if k == (LK.DENSE, LK.COMPRESSED) and fmt.levels[1].props.ordered:
            return "csr"
        if (k == (LK.COMPRESSED, LK.SINGLETON) and fmt.levels[0].props.ordered
                and fmt.levels[1].props.ordered):
            return "coo"
        if k == (LK.COMPRESSED, LK.SINGLETON, LK.SINGLETON) and all(
                s.props.ordered for s in fmt.levels):
            return "coo3"   # lexicographically sorted (an unordered level is Reordered)
        if k == (LK.COMPRESSED, LK.COMPRESSED, LK.COMPRESSED) and all(
                s.props.ordered and s.props.unique for s in fmt.levels):
            return "csf"
        if k == (LK.HASHED,):
            return "hash1"
        if k == (LK.HASHED, LK.DENSE):
            return "hash_dense"     # hashed rows over dense columns
        if k == (LK.DENSE, LK.HASHED):
            return "dense_hash"     # a hashed segment of columns per row
        if k == (LK.COMPRESSED,) and fmt.levels[0].props.ordered and fmt.levels[0].props.unique:
            return "spvec"
    roles = tuple(r.part for r in fmt.roles)
    if k == (LK.DENSE, LK.DENSE, LK.SINGLETON) and roles == ("slot", "whole", "whole"):
        return "ell"
    if k == (LK.DENSE, LK.RANGE, LK.OFFSET) and roles == ("diag", "whole", "whole"):
        return "dia"
    return "other:" + fmt.describe()


# ---------------------------------------------------------------------------
# plans

@dataclass
class Plan:
    pattern: str                 # spmv | add | mttkrp
    kernel: str                  # which C-ABI entry executes it
    operands: Dict[str, str]     # role -> tensor name
    out_format: TensorFormat
    out_dims: Tuple[int, ...]
    fuse: bool = True            # the reference's fuse_branchless switch (engine.py:766-772)
    out_class: str = ""          # format_class(out_format), fixed at planning
    ivars: Tuple[str, ...] = ()  # the loop variables, in schedule order (EvalStats keys)
    order: Tuple[str, ...] = ()  # tensor names in expression order (lattice-point labels)


def _flatten_mul(e):
    if isinstance(e, Mul):
        return _flatten_mul(e.left) + _flatten_mul(e.right)
    return [e]


def plan(checked: CheckedExpr, bindings, out_format: TensorFormat,
         out_dims: Tuple[int, ...], *, fuse: bool = True) -> Plan:
    """Bind the expression to a kernel (or raise).  `fuse` follows the
    reference's `plan(..., fuse=)` (engine.py:766-772): an unfused COO chain
    is executed level by level, so its duplicate coordinates are grouped
    (engine.py:200-209) — the B200 path then runs the exact-CSR copy."""
    p = _plan(checked, bindings, out_format, out_dims, fuse)
    p.fuse = fuse
    p.out_class = format_class(out_format)
    p.order = tuple(dict.fromkeys(t.tensor for t in _accesses(checked.assignment.rhs)))
    return p


def _accesses(e):
    if isinstance(e, Access):
        return [e]
    return _accesses(e.left) + _accesses(e.right) if isinstance(e, (Mul, Add)) else []


def _plan(checked: CheckedExpr, bindings, out_format: TensorFormat,
          out_dims: Tuple[int, ...], fuse: bool) -> Plan:
    a: Assignment = checked.assignment
    lhs, rhs = a.lhs, a.rhs
    cls = {name: format_class(fmt) for name, (fmt, _) in bindings.items()}
    ocls = format_class(out_format)

    # ---- SpMV: y(i) = A(i,j) * x(j)
    if isinstance(rhs, Mul) and all(isinstance(t, Access) for t in (rhs.left, rhs.right)):
        acc = [rhs.left, rhs.right]
        mat = [t for t in acc if len(t.ivars) == 2]
        vec = [t for t in acc if len(t.ivars) == 1]
        if len(mat) == 1 and len(vec) == 1 and len(lhs.ivars) == 1:
            A, x = mat[0], vec[0]
            i, j = A.ivars
            if lhs.ivars == (i,) and x.ivars == (j,) and i != j:
                if ocls not in ("dense1", "hash1"):
                    raise UnsupportedOutputError(
                        f"SpMV output must be a dense or hash vector, got {out_format.describe()}")
                ca, cx = cls[A.tensor], cls[x.tensor]
                kern = None
                if cx == "dense1" and ca in ("coo", "csr", "ell", "dia"):
                    kern = f"spmv_{ca}" if (fuse or ca != "coo") else "spmv_coo_grouped"
                elif cx == "hash1" and ca == "csr":
                    kern = "spmv_csr_hashx"
                elif cx == "spvec" and ca == "csr":
                    kern = "spmv_csr_spx"
                if kern is not None:
                    return Plan("spmv", kern, {"A": A.tensor, "x": x.tensor}, out_format,
                                out_dims, ivars=(i, j))
                raise UnsupportedMergeError(
                    f"no B200 kernel for SpMV with A {ca} and x {cx}")

    # ---- SpMM: Y(i,k) = A(i,j) * X(j,k), A CSR, X dense-2
    if isinstance(rhs, Mul) and all(isinstance(t, Access) for t in (rhs.left, rhs.right)):
        acc = [rhs.left, rhs.right]
        if all(len(t.ivars) == 2 for t in acc) and len(lhs.ivars) == 2:
            for A, X in ((acc[0], acc[1]), (acc[1], acc[0])):
                i, j = A.ivars
                if (X.ivars[0] == j and lhs.ivars == (i, X.ivars[1])
                        and len({i, j, X.ivars[1]}) == 3):
                    ca, cx = cls[A.tensor], cls[X.tensor]
                    if ca in ("csr", "coo") and cx == "dense2":
                        if ocls not in ("dense2", "hash_dense"):
                            raise UnsupportedOutputError(
                                "SpMM output must be dense-2 or {hashed, dense}")
                        kern = "spmm_csr" if ca == "csr" else (
                            "spmm_coo" if fuse else "spmm_coo_grouped")
                        return Plan("spmm", kern, {"A": A.tensor, "X": X.tensor},
                                    out_format, out_dims, ivars=(i, j, X.ivars[1]))
            raise UnsupportedMergeError("no B200 kernel for this matrix product "
                                        "(supported: CSR / COO x dense-2)")

    # ---- 3-tensor x vector / matrix / tensor (X CSF or COO-3)
    if isinstance(rhs, Mul) and all(isinstance(t, Access) for t in (rhs.left, rhs.right)):
        acc = [rhs.left, rhs.right]
        X3 = [t for t in acc if len(t.ivars) == 3]
        if len(X3) >= 1:
            X = X3[0]
            other = acc[1] if acc[0] is X else acc[0]
            i, j, k = X.ivars
            cX, cO = cls[X.tensor], cls[other.tensor]
            # TTV: Y(i,j) = X(i,j,k) * v(k)
            if other.ivars == (k,) and lhs.ivars == (i, j) and len({i, j, k}) == 3:
                if (cX == "csf" or (cX == "coo3" and fuse)) and cO == "dense1":
                    if ocls not in ("dense2", "csr"):
                        raise UnsupportedOutputError("TTV output must be dense-2 or CSR")
                    return Plan("ttv", f"ttv_{cX}_{ocls}", {"X": X.tensor, "v": other.tensor},
                                out_format, out_dims, ivars=(i, j, k))
                raise UnsupportedMergeError(f"no B200 kernel for TTV with X {cX}, v {cO}")
            # TTM: Y(i,j,r) = X(i,j,k) * U(k,r)
            if (len(other.ivars) == 2 and other.ivars[0] == k and len(lhs.ivars) == 3
                    and lhs.ivars == (i, j, other.ivars[1]) and len({i, j, k, other.ivars[1]}) == 4):
                if (cX == "csf" or (cX == "coo3" and fuse)) and cO == "dense2":
                    if ocls != "dense3":
                        raise UnsupportedOutputError("TTM output must be dense-3")
                    return Plan("ttm", f"ttm_{cX}", {"X": X.tensor, "U": other.tensor},
                                out_format, out_dims, ivars=(i, j, k, other.ivars[1]))
                raise UnsupportedMergeError(f"no B200 kernel for TTM with X {cX}, U {cO}")
            # INNERPROD: a() = X(i,j,k) * Z(i,j,k)
            if other.ivars == X.ivars and lhs.ivars == () and len({i, j, k}) == 3:
                if cX == "coo3" and cO == "coo3":
                    if ocls != "dense0":
                        raise UnsupportedOutputError("inner product output must be a scalar")
                    return Plan("inner", "inner_coo3", {"X": X.tensor, "Z": other.tensor},
                                out_format, out_dims, ivars=(i, j, k))
                raise UnsupportedMergeError(
                    f"no B200 kernel for the inner product of {cX} and {cO} (COO-3 x COO-3)")

    # ---- A(i,j,k) = X(i,j,k) + Z(i,j,k) (3rd-order PLUS): the union merge of
    # the (i,j)-fibre x k matrices — the 2-D A + B kernels over fibre keys
    if isinstance(rhs, Add) and all(isinstance(t, Access) for t in (rhs.left, rhs.right)):
        L_, R_ = rhs.left, rhs.right
        if len(lhs.ivars) == 3 and L_.ivars == lhs.ivars and R_.ivars == lhs.ivars and \
                len(set(lhs.ivars)) == 3:
            cl, cr = cls[L_.tensor], cls[R_.tensor]
            if cl in ("coo3", "csf") and cr in ("coo3", "csf"):
                if ocls not in ("coo3", "csf", "dense3"):
                    raise UnsupportedOutputError(
                        f"PLUS output must be COO-3, CSF or dense-3; got {out_format.describe()}")
                return Plan("plus3", f"plus3_{ocls}", {"X": L_.tensor, "Z": R_.tensor},
                            out_format, out_dims, ivars=lhs.ivars)
            raise UnsupportedMergeError(f"no B200 kernel for PLUS with {cl} + {cr}")

    # ---- C(i,j) = A(i,j) + B(i,j)
    if isinstance(rhs, Add) and all(isinstance(t, Access) for t in (rhs.left, rhs.right)):
        L_, R_ = rhs.left, rhs.right
        if len(lhs.ivars) == 2 and L_.ivars == lhs.ivars and R_.ivars == lhs.ivars:
            if ocls not in ("csr", "coo", "dense_hash"):
                raise UnsupportedOutputError(
                    f"A + B is assembled by gather-append into CSR or COO (or scattered into "
                    f"a hashed row segment); got {out_format.describe()}")
            cl, cr = cls[L_.tensor], cls[R_.tensor]
            if cl in ("csr", "coo") and cr in ("csr", "coo"):
                # a + b == b + a bit-for-bit: keep a CSR operand (if any) as A and
                # a COO one as B, whose duplicate coordinates the kernels group
                A_, B_ = (L_, R_) if (cl == "csr" or cr == "coo") else (R_, L_)
                ca = cls[A_.tensor]
                ko = "hash" if ocls == "dense_hash" else ocls
                return Plan("add", f"add_{ca}_{cls[B_.tensor]}_{ko}",
                            {"A": A_.tensor, "B": B_.tensor}, out_format, out_dims,
                            ivars=lhs.ivars)
            raise UnsupportedMergeError(f"no B200 kernel for A + B with {cl} + {cr}")

    # ---- A(i,r) = X(i,j,k) * B(j,r) * C(k,r), association (X*B)*C
    if isinstance(rhs, Mul) and len(_flatten_mul(rhs)) == 3 and all(
            isinstance(t, Access) for t in _flatten_mul(rhs)):
        inner, outer = (rhs.left, rhs.right) if isinstance(rhs.left, Mul) else (rhs.right,
                                                                                 rhs.left)
        if isinstance(inner, Mul) and isinstance(outer, Access):
            pair = [inner.left, inner.right]
            X = [t for t in pair if len(t.ivars) == 3]
            Bm = [t for t in pair if len(t.ivars) == 2]
            if len(X) == 1 and len(Bm) == 1 and len(outer.ivars) == 2:
                X, Bm, Cm = X[0], Bm[0], outer
                i, j, k = X.ivars
                if (len({i, j, k}) == 3 and len(lhs.ivars) == 2 and lhs.ivars[0] == i
                        and Bm.ivars == (j, lhs.ivars[1]) and Cm.ivars == (k, lhs.ivars[1])):
                    if ocls not in ("dense2", "hash_dense"):
                        raise UnsupportedOutputError(
                            "MTTKRP output must be dense-2 or {hashed, dense}")
                    cX = cls[X.tensor]
                    if cX in ("coo3", "csf") and cls[Bm.tensor] == "dense2" and \
                            cls[Cm.tensor] == "dense2":
                        return Plan("mttkrp", f"mttkrp_{cX}",
                                    {"X": X.tensor, "B": Bm.tensor, "C": Cm.tensor},
                                    out_format, out_dims, ivars=(i, j, k, lhs.ivars[1]))
                    raise UnsupportedMergeError(
                        f"no B200 kernel for MTTKRP with X {cX}, B {cls[Bm.tensor]}, "
                        f"C {cls[Cm.tensor]}")
    raise UnsupportedMergeError(
        "no B200 kernel implements this expression/format combination "
        "(supported: SpMV over coo/csr/ell/dia with dense x, CSR with hashed or sparse-vector x, "
        "SpMM CSR x dense-2, CSR + COO/CSR -> CSR, MTTKRP over COO-3/CSF, TTV/TTM over CSF, "
        "inner product of COO-3 tensors)")


# ---------------------------------------------------------------------------
# execution

def _dev(st: TensorStorage, device):
    if st.vals.device != device:
        return st.to(device, non_blocking=True)
    return st


def _dia_host_offsets(st: TensorStorage):
    offs = getattr(st, "_host_offsets", None)
    if offs is None:
        offs = st.levels[1].offset.cpu().numpy().astype(np.int32)
        st._host_offsets = offs
    return offs


def _dense_level(spec, n: int) -> LevelStorage:
    """A dense output level (no arrays): built without the array conversions
    of LevelStorage.__init__ — the e2e step pays this per call."""
    lv = LevelStorage.__new__(LevelStorage)
    lv.spec, lv.n, lv.m, lv.w = spec, int(n), 0, 0
    lv.pos = lv.crd = lv.offset = None
    lv.crd_stride, lv.crd_base, lv.range_n = 1, 0, 0
    lv._appended = lv._edges = None
    lv._last_edge_parent = -1
    lv._sl_max_row = None
    return lv


def _hashed_row_order(p: Plan, A: TensorStorage, nrows: int, dev):
    """Row coordinates in the order the reference's scatter writer first
    writes them (engine.py:281-327): CSR writes every row's total after its
    loop (empty rows included); COO one write per nonzero (present rows, in
    storage order); ELL every row once per slot (no rows when there are no
    slots); DIA the rows of each diagonal's range [max(0,-o), min(n, m-o))
    (levels.py:220-222), diagonal by diagonal in offset order.  The ordered
    insert keeps each coordinate's first occurrence."""
    if p.kernel in ("spmv_coo", "spmv_coo_grouped"):
        return torch.unique_consecutive(A.levels[0].crd)
    if p.kernel == "spmv_ell":
        if A.levels[0].n == 0:
            return torch.empty(0, dtype=torch.int32, device=dev)
        return torch.arange(nrows, dtype=torch.int32, device=dev)
    if p.kernel == "spmv_dia":
        ncols = A.dims[1]
        parts = [torch.arange(max(0, -o), min(nrows, ncols - o), dtype=torch.int32, device=dev)
                 for o in _dia_host_offsets(A).tolist()]
        return torch.cat(parts) if parts else torch.empty(0, dtype=torch.int32, device=dev)
    return torch.arange(nrows, dtype=torch.int32, device=dev)


def _hashed_spmv_output(p: Plan, A: TensorStorage, y, nrows: int, dev) -> TensorStorage:
    """SpMV into a hash-vector output, as the reference's scatter writer builds
    it (engine.py:281-327): the row coordinates are inserted in the order
    they are first written (`_hashed_row_order`) and each slot holds the
    row's sum, which is the dense kernel's y[i] (the same additions from
    +0.0).  Width: the format's pinned width, else next_pow2(max(4, 2 n))."""
    f = p.out_format
    w = f.hash_width or _next_pow2(max(4, 2 * nrows))
    rows = _hashed_row_order(p, A, nrows, dev)
    crd, err = K.hashed_insert(rows, w)
    if int(err.item()) != 0:
        raise HashSegmentFullError(f"hashed segment of width {w} is full")
    vals = torch.zeros(w, dtype=torch.float64, device=dev)
    if rows.numel():
        slots, _ = K.hashed_locate(rows, w, crd)
        vals[slots.long()] = y[rows.long()]
    return TensorStorage(f, (nrows,), [LevelStorage(f.levels[0], w=w, crd=crd, device=dev)], vals)


def _csr_level(st: TensorStorage):
    """(compressed level, vals) of a {dense, compressed} matrix with one entry per
    coordinate.  A non-unique compressed level is iterated through the
    reference's `Grouped` (engine.py:107-149, 200-209): each run of equal
    coordinates is one visit whose value is the run's sum (engine.py:520-527)
    — the exact identity copy (gather-append, 0.0 + (v1 + v2 ...)) is that
    matrix, bit for bit where it can matter (a lone -0.0 group only feeds
    sums that start from +0.0).  Computed once per storage and cached."""
    lv = st.levels[1]
    if st.format.levels[1].props.unique:
        return lv, st.vals
    cached = getattr(st, "_sl_grouped", None)
    if cached is None or cached[0] is not lv.pos:
        nrows = st.dims[0]
        empty_i = torch.empty(0, dtype=torch.int32, device=lv.pos.device)
        a_pos = torch.zeros(nrows + 1, dtype=torch.int32, device=lv.pos.device)
        pos, crd, vals = K.add_csr(nrows, a_pos, empty_i, empty_i.double(), lv.crd, st.vals,
                                   b_pos=lv.pos)
        cached = (lv.pos, LevelStorage(lv.spec, pos=pos, crd=crd, device=pos.device), vals)
        st._sl_grouped = cached
    return cached[1], cached[2]


def _csr_arrays(st: TensorStorage):
    lv, vals = _csr_level(st)
    return lv.pos, lv.crd, vals


def _hashed_rows_output(f: TensorFormat, dims, rows, Y, dev) -> TensorStorage:
    """{hashed, dense} output of a row-scattered result Y (rows x cols, dense):
    the written rows inserted in first-write order (the ordered bulk insert
    = the reference's sequential insert_coord calls, levels.py:312-333), each
    slot holding its row (engine.py:292-317)."""
    n, ncols = dims
    w = f.hash_width or _next_pow2(max(4, 2 * n))
    crd, err = K.hashed_insert(rows, w)
    if int(err.item()) != 0:
        raise HashSegmentFullError(f"hashed segment of width {w} is full")
    vals = torch.zeros(w * ncols, dtype=torch.float64, device=dev)
    if rows.numel():
        slots, _ = K.hashed_locate(rows, w, crd)
        vals.view(w, ncols)[slots.long()] = Y.reshape(n, ncols)[rows.long()]
    return TensorStorage(f, tuple(dims), [LevelStorage(f.levels[0], w=w, crd=crd, device=dev),
                                          LevelStorage(f.levels[1], n=ncols, device=dev)], vals)


def _hashed_segments_output(f: TensorFormat, dims, c_pos, c_crd, c_vals, dev) -> TensorStorage:
    """{dense, hashed} output of a row-wise union (A + B): row i's columns
    inserted into segment i in ascending order (the order the gather of the
    union writes them), each slot holding its value."""
    n, ncols = dims
    w = f.hash_width or _next_pow2(max(4, 2 * ncols))
    nnz = int(c_crd.numel())
    rows = K.csr_rows(n, c_pos, nnz)
    crd, err = K.hashed_insert(c_crd, w, nseg=max(n, 1), parent=rows)
    if int(err.item()) != 0:
        raise HashSegmentFullError(f"hashed segment of width {w} is full")
    vals = torch.zeros(max(n, 1) * w, dtype=torch.float64, device=dev)
    if nnz:
        slots, _ = K.hashed_locate(c_crd, w, crd, parent=rows)
        vals[slots.long()] = c_vals
    return TensorStorage(f, tuple(dims), [LevelStorage(f.levels[0], n=n, device=dev),
                                          LevelStorage(f.levels[1], w=w, crd=crd, device=dev)],
                         vals)


def _coo3_fibres(X: TensorStorage):
    """The (i, j)-fibre structure of an ordered COO-3 as CSF-shaped levels
    (slices, fibres, leaves), derived on the device from the coordinates
    (the leaves are X's own k coordinates and values, duplicates kept)."""
    i, j, k = X.levels[0].crd, X.levels[1].crd, X.levels[2].crd
    dev = k.device
    nnz = int(k.numel())
    if nnz == 0:
        z = torch.zeros(1, dtype=torch.int32, device=dev)
        e = torch.empty(0, dtype=torch.int32, device=dev)
        return [LevelStorage(X.levels[0].spec, crd=e, device=dev),
                LevelStorage(X.levels[1].spec, pos=z, crd=e, device=dev),
                LevelStorage(X.levels[2].spec, pos=z, crd=k, device=dev)]
    J = X.dims[1]
    key = i.to(torch.int64) * J + j.to(torch.int64)
    fst = torch.ones(nnz, dtype=torch.bool, device=dev)
    fst[1:] = key[1:] != key[:-1]
    fpos = torch.nonzero(fst).squeeze(1)
    fi = i[fpos]
    sst = torch.ones(fpos.numel(), dtype=torch.bool, device=dev)
    sst[1:] = fi[1:] != fi[:-1]
    spos = torch.nonzero(sst).squeeze(1)
    end = lambda t, v: torch.cat([t, torch.tensor([v], device=dev)]).to(torch.int32)  # noqa: E731
    return [LevelStorage(X.levels[0].spec, crd=fi[spos], device=dev),
            LevelStorage(X.levels[1].spec, pos=end(spos, fpos.numel()), crd=j[fpos], device=dev),
            LevelStorage(X.levels[2].spec, pos=end(fpos, nnz), crd=k, device=dev)]


def _coo3_grouped(X: TensorStorage):
    """CSF-shaped levels and values of a COO-3 whose repeated (i, j, k) are
    grouped (Grouped, engine.py:107-149: one visit, Python's sum() of the
    run): the exact copy of the (fibre x k) matrix whose rows are X's
    distinct fibres (keys i*J + j, located by searchsorted)."""
    I, J, Kd = X.dims
    key, kc, v = _fibre_coo(X)
    fk = torch.unique_consecutive(key) if key.numel() else key
    rows = torch.searchsorted(fk, key).to(torch.int32)
    pos, crd, vals = K.coo_to_csr(int(fk.numel()), rows, kc, v)
    dev = vals.device
    fi = (fk // J).to(torch.int32)
    sst = torch.ones(fk.numel(), dtype=torch.bool, device=dev)
    if fk.numel():
        sst[1:] = fi[1:] != fi[:-1]
    spos = torch.nonzero(sst).squeeze(1)
    end = lambda t, n: torch.cat([t.to(torch.int64), torch.tensor([n], device=dev)]).to(  # noqa: E731
        torch.int32)
    return [LevelStorage(X.levels[0].spec, crd=fi[spos], device=dev),
            LevelStorage(X.levels[1].spec, pos=end(spos, fk.numel()),
                         crd=(fk % J).to(torch.int32), device=dev),
            LevelStorage(X.levels[2].spec, pos=pos, crd=crd, device=dev)], vals


def _fibre_coo(X: TensorStorage, narrow: bool = False):
    """(fibre key i*J + j, k, vals) of a COO-3 or CSF operand, in storage
    order.  Keys are int64; with `narrow`, int32 when I*J fits (half the
    traffic of every pass over the keys)."""
    I, J = X.dims[0], X.dims[1]
    kt = torch.int32 if narrow and I * J <= 2 ** 31 - 1 else torch.int64
    if format_class(X.format) == "coo3":
        key = X.levels[0].crd.to(kt) * J + X.levels[1].crd.to(kt)
        return key, X.levels[2].crd, X.vals[:X.levels[2].crd.numel()]
    if kt is torch.int32:
        key, kc, v = _fibre_coo(X)
        return key.to(kt), kc, v
    L = X.levels
    n1 = int(L[1].crd.numel())
    nnz = int(L[2].crd.numel())
    dev = X.vals.device
    fs = torch.repeat_interleave(torch.arange(L[0].crd.numel(), device=dev),
                                 (L[1].pos[1:] - L[1].pos[:-1]).to(torch.int64))
    fkey = L[0].crd.to(torch.int64)[fs] * J + L[1].crd.to(torch.int64)
    leaf_f = torch.repeat_interleave(torch.arange(n1, device=dev),
                                     (L[2].pos[1:] - L[2].pos[:-1]).to(torch.int64))
    return fkey[leaf_f], L[2].crd, X.vals[:nnz]


_PLUS3_ROW = 16    # target entries per row of the 2-D union (a dense fibre is cut into k-blocks)


def _plus3(p: Plan, X: TensorStorage, Z: TensorStorage, dev) -> TensorStorage:
    """A(i,j,k) = X(i,j,k) + Z(i,j,k) as a 2-D union: the same gather-append
    and duplicate grouping as A + B (X's exact grouped copy, Z's repeats
    grouped by the kernels; engine.py:107-149, 330-434) with columns k and
    rows the union of the operands' (i, j) fibres (sorted keys i*J + j, each
    nonzero's fibre located by searchsorted) — a fibre holding many entries
    cut into power-of-two k-blocks of ~_PLUS3_ROW entries, each block its own
    row.  The union over (fibre, k-block, k) is the union over (i, j, k); what
    changes is the kernels' load balance: D5's power-law fibres (up to K
    entries each) as single rows serialised the long-row path (22.8 ms of
    A + B; k-blocked: see DESIGN.md)."""
    I, J, Kd = X.dims
    xk, xc, xv = _fibre_coo(X, narrow=True)
    zk, zc, zv = _fibre_coo(Z, narrow=True)
    uq = lambda t: torch.unique_consecutive(t) if t.numel() else t  # noqa: E731
    U = torch.unique(torch.cat([uq(xk), uq(zk)]))                   # sorted fibre keys
    nU = int(U.numel())
    xf = torch.searchsorted(U, xk, out_int32=True)
    zf = torch.searchsorted(U, zk, out_int32=True)
    if nU:
        # entries per union fibre: the keys are sorted, so two boundary searches
        # (a bincount's atomics pile up on the long fibres: 4 ms at D5)
        ub = torch.cat([U, U[-1:] + 1])       # (a narrow key is at most 2^31 - 2)
        ln = torch.diff(torch.searchsorted(xk, ub)) + torch.diff(torch.searchsorted(zk, ub))
        kbits = max(int(Kd) - 1, 1).bit_length()
        want = torch.ceil(torch.log2((ln.double() / _PLUS3_ROW).clamp_(min=1.0))).to(torch.int64)
        sh = (kbits - want).clamp_(min=0)                # k >> sh: the k-block of a coordinate
        nblk = ((Kd - 1) >> sh) + 1                      # rows of each fibre
        rowend = torch.cumsum(nblk, 0)
        rowbase = rowend - nblk
        nR = int(rowend[-1].item())
    else:
        sh = rowbase = nblk = torch.zeros(0, dtype=torch.int64, device=dev)
        nR = 0
    if nR > 2 ** 31 - 1:
        raise UnsupportedMergeError("3rd-order PLUS: the union's row space exceeds int32")
    rb32, sh32 = rowbase.to(torch.int32), sh.to(torch.int32)
    xr = rb32[xf] + (xc >> sh32[xf])
    zr = rb32[zf] + (zc >> sh32[zf])
    a_pos, a_crd, a_vals = K.coo_to_csr(nR, xr, xc, xv)
    c_pos, c_crd, c_vals = K.add_csr(nR, a_pos, a_crd, a_vals, zc, zv, b_rows=zr)
    f = p.out_format
    ocls = format_class(f)
    nnz = int(c_crd.numel())
    fi, fj = (U // J).to(torch.int32), (U % J).to(torch.int32)

    def out_fibres():       # union fibre of every output entry
        rowfib = torch.repeat_interleave(torch.arange(nU, dtype=torch.int32, device=dev), nblk)
        return rowfib[K.csr_rows(nR, c_pos, nnz)]

    if ocls == "dense3":
        out = torch.zeros(I * J * Kd, dtype=torch.float64, device=dev)
        if nnz:
            out[U.to(torch.int64)[out_fibres()] * Kd + c_crd.to(torch.int64)] = c_vals
        return TensorStorage(f, (I, J, Kd), [LevelStorage(s_, n=d, device=dev)
                                             for s_, d in zip(f.levels, (I, J, Kd))], out)
    if ocls == "coo3":
        fib = out_fibres() if nnz else torch.empty(0, dtype=torch.int32, device=dev)
        return TensorStorage(f, (I, J, Kd), [LevelStorage(f.levels[0], pos=[0, nnz], crd=fi[fib],
                                                          device=dev),
                                             LevelStorage(f.levels[1], crd=fj[fib], device=dev),
                                             LevelStorage(f.levels[2], crd=c_crd, device=dev)],
                             c_vals)
    # CSF: every union fibre holds an entry; slices are the runs of equal i;
    # a fibre's leaves are its k-blocks' rows, consecutive in C
    sst = torch.ones(nU, dtype=torch.bool, device=dev)
    if nU:
        sst[1:] = fi[1:] != fi[:-1]
    spos = torch.nonzero(sst).squeeze(1)
    end = lambda t, v: torch.cat([t.to(torch.int64), torch.tensor([v], device=dev)]).to(  # noqa: E731
        torch.int32)
    leaf_pos = c_pos[end(rowbase, nR).to(torch.int64)] if nU else c_pos
    return TensorStorage(f, (I, J, Kd), [
        LevelStorage(f.levels[0], pos=[0, int(spos.numel())], crd=fi[spos], device=dev),
        LevelStorage(f.levels[1], pos=end(spos, nU), crd=fj, device=dev),
        LevelStorage(f.levels[2], pos=leaf_pos, crd=c_crd, device=dev)], c_vals)


_SKEW_TILE = 4 * 896   # 32-row tiles heavier than four hand-off stages: merge-path


def _csr_variant(lv: LevelStorage) -> int:
    """CSR SpMV variant for this matrix: the automatic choice (register
    hand-off for short rows, row-block otherwise), or the merge-path split when
    some 32-row tile holds more than four hand-off stages of nonzeros —
    power-law rows otherwise serialise one persistent warp per heavy tile
    (D5's fibres: 2.6 ms vs 0.23 ms).  The heaviest tile is measured once per
    row-pointer array and cached on the level."""
    return 2 if _row_stats(lv)[0] > _SKEW_TILE else 0


def _row_stats(lv: LevelStorage):
    """(heaviest 32-row tile, longest row) of a compressed level, measured once
    per row-pointer array and cached on the level."""
    cached = lv._sl_max_row
    if cached is None or cached[0] is not lv.pos:
        pos = lv.pos
        n = pos.numel() - 1
        if n > 0:
            idx = torch.arange(0, n + 32, 32, device=pos.device).clamp_(max=n)
            tb = pos[idx].to(torch.int64)
            both = torch.stack([(tb[1:] - tb[:-1]).max(), (pos[1:] - pos[:-1]).max().long()])
            heaviest, longest = (int(v) for v in both.tolist())
        else:
            heaviest = longest = 0
        cached = (pos, heaviest, longest)
        lv._sl_max_row = cached
    return cached[1], cached[2]


_SPMM_LONG_ROW = 1024  # SpMM rows longer than this: one CTA per row (power-law rows)


def _next_pow2(v: int) -> int:
    n = 1
    while n < v:
        n <<= 1
    return n


def _run(p: Plan, inputs: Dict[str, TensorStorage], stats: Optional[EvalStats]):
    dev = None
    for st in inputs.values():
        if st.vals.is_cuda:
            dev = st.vals.device
            break
    if dev is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if dev.index is not None and dev.index != torch._C._cuda_getDevice():
        # kernels launch on the current device's current stream: make it the
        # operands' device for the call (outputs are allocated there too)
        with torch.cuda.device(dev):
            return _run_on(p, inputs, stats, dev)
    return _run_on(p, inputs, stats, dev)


def _run_on(p: Plan, inputs: Dict[str, TensorStorage], stats: Optional[EvalStats], dev):
    ops = {role: _dev(inputs[name], dev) for role, name in p.operands.items()}

    if p.pattern == "spmv":
        A, x = ops["A"], ops["x"]
        nrows, ncols = A.dims
        if p.kernel == "spmv_coo":
            y = K.spmv_coo(nrows, ncols, A.levels[0].crd, A.levels[1].crd, A.vals, x.vals)
        elif p.kernel == "spmv_coo_grouped":
            # unfused COO: rows and (row, column) runs grouped — the exact CSR copy
            pos, crd, vals = K.coo_to_csr(nrows, A.levels[0].crd, A.levels[1].crd, A.vals)
            y = K.spmv_csr(nrows, ncols, pos, crd, vals, x.vals)
        elif p.kernel == "spmv_csr":
            lv, vals = _csr_level(A)
            y = K.spmv_csr(nrows, ncols, lv.pos, lv.crd, vals, x.vals, variant=_csr_variant(lv))
        elif p.kernel == "spmv_ell":
            S = A.levels[0].n
            y = K.spmv_ell(nrows, ncols, S, A.levels[2].crd, A.vals, x.vals)
        elif p.kernel == "spmv_dia":
            offs = _dia_host_offsets(inputs[p.operands["A"]])
            if len(offs) > 32:   # beyond the kernel-parameter window: the level's device array
                offs = A.levels[1].offset
            y = K.spmv_dia(nrows, ncols, offs, A.vals, x.vals)
        elif p.kernel == "spmv_csr_spx":
            sx = x.levels[0]
            pos, crd, vals = _csr_arrays(A)
            y = K.spmv_csr_spx(nrows, int(x.dims[0]), pos, crd, vals, sx.crd, x.vals)
        else:  # spmv_csr_hashx
            hx = x.levels[0]
            pos, crd, vals = _csr_arrays(A)
            nq = int(crd.numel())
            # queries >= table slots: resolve each coordinate once (slot map)
            n_map = int(x.dims[0]) if nq >= hx.w else None
            y = K.spmv_csr_hashx(nrows, pos, crd, vals, hx.w, hx.crd, x.vals, n=n_map)
        if p.out_class == "hash1":
            out = _hashed_spmv_output(p, A, y, nrows, dev)
        else:
            out = TensorStorage(p.out_format, (nrows,), [_dense_level(p.out_format.levels[0], nrows)],
                                y)
    elif p.pattern == "add":
        A, B = ops["A"], ops["B"]
        nrows = A.dims[0]
        _, ka, kb, ko = p.kernel.split("_")
        if ka == "coo":          # COO A (possibly duplicated): its exact CSR copy
            a_pos, a_crd, a_vals = K.coo_to_csr(nrows, A.levels[0].crd, A.levels[1].crd, A.vals)
        else:                    # CSR A, a non-unique level grouped
            a_pos, a_crd, a_vals = _csr_arrays(A)
        if kb == "coo":
            c_pos, c_crd, c_vals = K.add_csr(nrows, a_pos, a_crd, a_vals, B.levels[1].crd, B.vals,
                                             b_rows=B.levels[0].crd)
        else:
            c_pos, c_crd, c_vals = K.add_csr(nrows, a_pos, a_crd, a_vals, B.levels[1].crd, B.vals,
                                             b_pos=B.levels[1].pos)
        f = p.out_format
        if ko == "csr":
            out = TensorStorage(f, A.dims, [LevelStorage(f.levels[0], n=nrows, device=dev),
                                            LevelStorage(f.levels[1], pos=c_pos, crd=c_crd,
                                                         device=dev)], c_vals)
        elif ko == "hash":           # dense_hash: each row's columns in its own segment
            out = _hashed_segments_output(f, A.dims, c_pos, c_crd, c_vals, dev)
        else:
            rows = K.csr_rows(nrows, c_pos, c_crd.numel())
            nnz = int(c_crd.numel())
            out = TensorStorage(f, A.dims, [LevelStorage(f.levels[0], pos=[0, nnz], crd=rows,
                                                         device=dev),
                                            LevelStorage(f.levels[1], crd=c_crd, device=dev)],
                                c_vals)
        res_csr = (c_pos, c_crd)
    elif p.pattern == "spmm":
        A, X = ops["A"], ops["X"]
        nrows, ncols = A.dims
        Kc = X.dims[1]
        if p.kernel == "spmm_coo":           # fused COO chain: the row level's position index
            lv = LevelStorage(A.levels[0].spec, pos=K.coo_rowptr(nrows, A.levels[0].crd),
                              crd=A.levels[1].crd, device=dev)
            vals = A.vals
        elif p.kernel == "spmm_coo_grouped":  # unfused: rows and (row, column) runs grouped
            pos, crd, vals = K.coo_to_csr(nrows, A.levels[0].crd, A.levels[1].crd, A.vals)
            lv = LevelStorage(A.levels[1].spec, pos=pos, crd=crd, device=dev)
        else:
            lv, vals = _csr_level(A)
        long_min = _SPMM_LONG_ROW if _row_stats(lv)[1] > _SPMM_LONG_ROW else None
        Y = K.spmm_csr(nrows, ncols, lv.pos, lv.crd, vals, X.vals.view(ncols, Kc),
                       long_min=long_min)
        f = p.out_format
        if format_class(f) == "hash_dense":   # rows written = rows holding a nonzero
            cnt = lv.pos[1:] - lv.pos[:-1]
            rows = torch.nonzero(cnt > 0).squeeze(1).to(torch.int32)
            out = _hashed_rows_output(f, (nrows, Kc), rows, Y, dev)
        else:
            out = TensorStorage(f, (nrows, Kc), [LevelStorage(f.levels[0], n=nrows, device=dev),
                                                 LevelStorage(f.levels[1], n=Kc, device=dev)],
                                Y.reshape(-1))
    elif p.pattern in ("ttv", "ttm"):
        X = ops["X"]
        I, J, Kd = X.dims
        xv = X.vals
        if p.kernel == "ttv_coo3_csr":       # gather output: the chain's repeats grouped
            lv, xv = _coo3_grouped(X)
        elif "_coo3" in p.kernel:            # scatter output: per-nonzero, storage order
            lv = _coo3_fibres(X)
        else:
            lv = X.levels
        args = (I, J, Kd, lv[0].crd, lv[1].pos, lv[1].crd, lv[2].pos, lv[2].crd, xv)
        f = p.out_format
        if p.kernel.endswith("_csr"):
            pos, crd, vals = K.ttv_csf(*args, ops["v"].vals, out="csr")
            out = TensorStorage(f, (I, J), [LevelStorage(f.levels[0], n=I, device=dev),
                                            LevelStorage(f.levels[1], pos=pos, crd=crd,
                                                         device=dev)], vals)
        elif p.kernel.endswith("_dense2"):
            Y = K.ttv_csf(*args, ops["v"].vals)
            out = TensorStorage(f, (I, J), [LevelStorage(f.levels[0], n=I, device=dev),
                                            LevelStorage(f.levels[1], n=J, device=dev)],
                                Y.reshape(-1))
        else:
            U = ops["U"]
            R = U.dims[1]
            long_min = _SPMM_LONG_ROW if _row_stats(lv[2])[1] > _SPMM_LONG_ROW else None
            Y = K.ttm_csf(*args, U.vals.view(Kd, R), long_min=long_min)
            out = TensorStorage(f, (I, J, R), [LevelStorage(f.levels[0], n=I, device=dev),
                                               LevelStorage(f.levels[1], n=J, device=dev),
                                               LevelStorage(f.levels[2], n=R, device=dev)],
                                Y.reshape(-1))
    elif p.pattern == "plus3":
        out = _plus3(p, ops["X"], ops["Z"], dev)
    elif p.pattern == "inner":
        X, Z = ops["X"], ops["Z"]
        I, J, Kd = X.dims
        xs = (X.levels[0].crd, X.levels[1].crd, X.levels[2].crd, X.vals)
        zs = (Z.levels[0].crd, Z.levels[1].crd, Z.levels[2].crd, Z.vals)
        a = K.inner_coo3(I, J, Kd, xs, zs)
        out = TensorStorage(p.out_format, (), [], a)
    else:  # mttkrp
        X, B, C = ops["X"], ops["B"], ops["C"]
        I, J, Kd = X.dims
        R = B.dims[1]
        Bt, Ct = B.vals.view(J, R), C.vals.view(Kd, R)
        if p.kernel == "mttkrp_coo3":
            A = K.mttkrp_coo3(I, J, Kd, X.levels[0].crd, X.levels[1].crd, X.levels[2].crd,
                              X.vals, Bt, Ct)
        else:
            A = K.mttkrp_csf(I, J, Kd, X.levels[0].crd, X.levels[1].pos, X.levels[1].crd,
                             X.levels[2].pos, X.levels[2].crd, X.vals, Bt, Ct)
        f = p.out_format
        if format_class(f) == "hash_dense":   # rows written = the stored slices, in order
            rows = torch.unique_consecutive(X.levels[0].crd) if X.levels[0].crd.numel() else \
                X.levels[0].crd
            out = _hashed_rows_output(f, (I, R), rows, A, dev)
        else:
            out = TensorStorage(f, (I, R), [LevelStorage(f.levels[0], n=I, device=dev),
                                            LevelStorage(f.levels[1], n=R, device=dev)],
                                A.reshape(-1))
    if stats is not None:
        for (var, label), n in _loop_counts(p, ops, locals().get("res_csr")).items():
            if n:
                stats.count(var, label, n)
    return out


# ---------------------------------------------------------------------------
# EvalStats: the reference's loop-visit counts, keyed (variable, lattice point)

def _label(p: Plan, *dims: Tuple[str, int]) -> str:
    """Lattice-point label as the reference prints it (engine.py:255-268):
    `{A1,x0}` — each iterated or located tensor level, tensors in expression
    order."""
    rank = {t: n for n, t in enumerate(p.order)}
    ds = sorted(dims, key=lambda d: (rank.get(d[0], 99), d[1]))
    return "{" + ",".join(f"{t}{lvl}" for t, lvl in ds) + "}"


def _i64(t):
    return t.to(torch.int64)


def _merge_counts(ka, kb, w: int):
    """Visits of `merge_visits` (engine.py:211-225) over two ordered unique
    coordinate streams under each parent, for keys parent*w + coord (sorted,
    unique): (visits while both streams are live, visits of A's remainder,
    visits of B's remainder, keys present in both)."""
    u = torch.unique(torch.cat([ka, kb]))
    if u.numel() == 0:
        z = torch.zeros((), dtype=torch.int64, device=u.device)
        return z, z, z, u
    pu, cu = torch.div(u, w, rounding_mode="floor"), u % w

    def last(k):
        if k.numel() == 0:
            return torch.full_like(u, -1)
        ix = torch.searchsorted(k, (pu + 1) * w) - 1
        kk = k[ix.clamp(min=0)]
        ok = (ix >= 0) & (torch.div(kk, w, rounding_mode="floor") == pu)
        return torch.where(ok, kk % w, torch.full_like(kk, -1))

    la, lb = last(ka), last(kb)
    both = (la >= 0) & (lb >= 0) & (cu <= torch.minimum(la, lb))
    rest = ~both
    a_rest = rest & (la > lb)
    common = ka[torch.isin(ka, kb)] if ka.numel() and kb.numel() else ka[:0]
    return both.sum(), a_rest.sum(), (rest & ~(la > lb)).sum(), common


def _grouped_keys(rows, cols, w: int):
    """Sorted unique keys row*w + col of an ordered coordinate list."""
    if rows.numel() == 0:
        return torch.empty(0, dtype=torch.int64, device=rows.device)
    return torch.unique_consecutive(_i64(rows) * w + _i64(cols))


def _csr_keys(pos, crd, w: int):
    nrows = pos.numel() - 1
    rows = torch.repeat_interleave(torch.arange(nrows, device=pos.device),
                                   _i64(pos[1:] - pos[:-1]))
    return _grouped_keys(rows, crd[: rows.numel()], w)


def _loop_counts(p: Plan, ops, res_csr) -> Dict[Tuple[str, str], int]:
    """Per (loop variable, lattice point) visit counts of the reference's
    schedule for this plan (engine.py:255-268, 607-608, 688-689), from the
    storage sizes and, for merged streams, the coordinates themselves."""
    v = p.ivars
    n = {role: name for role, name in p.operands.items()}
    out: Dict[Tuple[str, str], int] = {}
    if p.pattern == "spmv":
        A, x = ops["A"], ops["x"]
        An, xn = n["A"], n["x"]
        nrows, ncols = A.dims
        if p.kernel == "spmv_coo":
            out[(v[0], _label(p, (An, 0)))] = int(A.levels[1].crd.numel())
        elif p.kernel == "spmv_coo_grouped":
            r, c = A.levels[0].crd, A.levels[1].crd
            out[(v[0], _label(p, (An, 0)))] = int(torch.unique_consecutive(r).numel()) \
                if r.numel() else 0
            out[(v[1], _label(p, (An, 1), (xn, 0)))] = int(_grouped_keys(r, c, ncols).numel())
        elif p.kernel == "spmv_ell":
            S = A.levels[0].n
            out[("slot$" + An + "0", _label(p, (An, 0)))] = S
            out[(v[0], _label(p, (An, 1)))] = S * nrows
            if not p.fuse:
                out[(v[1], _label(p, (An, 2), (xn, 0)))] = S * nrows
        elif p.kernel == "spmv_dia":
            offs = _dia_host_offsets(A).tolist()
            inr = sum(max(0, min(nrows, ncols - o) - max(0, -o)) for o in offs)
            out[("diag$" + An + "0", _label(p, (An, 0)))] = len(offs)
            out[(v[0], _label(p, (An, 1)))] = inr
            if not p.fuse:
                out[(v[1], _label(p, (An, 2), (xn, 0)))] = inr
        else:                                   # CSR rows, grouped columns
            lv, _ = _csr_level(A)
            out[(v[0], _label(p, (An, 0)))] = nrows
            jl = _label(p, (An, 1), (xn, 0))
            if p.kernel == "spmv_csr_spx":      # intersection with x's stream
                out[(v[1], jl)] = _spx_visits(lv.pos, lv.crd, x.levels[0].crd)
            else:
                out[(v[1], jl)] = int(lv.crd.numel())
    elif p.pattern == "spmm":
        A, X = ops["A"], ops["X"]
        Kc = X.dims[1]
        if p.kernel == "spmm_coo":            # fused chain: one visit per nonzero
            nnz = int(A.levels[1].crd.numel())
            out[(v[0], _label(p, (n["A"], 0)))] = nnz
            out[(v[2], _label(p, (n["X"], 1)))] = nnz * Kc
        elif p.kernel == "spmm_coo_grouped":
            r, c = A.levels[0].crd, A.levels[1].crd
            nr = int(torch.unique_consecutive(r).numel()) if r.numel() else 0
            nij = int(_grouped_keys(r, c, A.dims[1]).numel())
            out[(v[0], _label(p, (n["A"], 0)))] = nr
            out[(v[1], _label(p, (n["A"], 1), (n["X"], 0)))] = nij
            out[(v[2], _label(p, (n["X"], 1)))] = nij * Kc
        else:
            lv, _ = _csr_level(A)
            nnz = int(lv.crd.numel())
            out[(v[0], _label(p, (n["A"], 0)))] = A.dims[0]
            out[(v[1], _label(p, (n["A"], 1), (n["X"], 0)))] = nnz
            out[(v[2], _label(p, (n["X"], 1)))] = nnz * Kc
    elif p.pattern == "add":
        out.update(_add_counts(p, ops, res_csr))
    elif p.pattern == "mttkrp":
        X, R = ops["X"], ops["B"].dims[1]
        Xn, Bn, Cn = n["X"], n["B"], n["C"]
        nnz = int(X.levels[-1].crd.numel()) if X.vals.numel() else 0
        if p.kernel == "mttkrp_coo3" and p.fuse:
            out[(v[0], _label(p, (Xn, 0)))] = nnz
            out[(v[3], _label(p, (Bn, 1), (Cn, 1)))] = nnz * R
        else:
            ni, nij, nijk = _coo3_level_sizes(X) if p.kernel == "mttkrp_coo3" else (
                int(X.levels[0].crd.numel()), int(X.levels[1].crd.numel()), nnz)
            out[(v[0], _label(p, (Xn, 0)))] = ni
            out[(v[1], _label(p, (Xn, 1), (Bn, 0)))] = nij
            out[(v[2], _label(p, (Xn, 2), (Cn, 0)))] = nijk
            out[(v[3], _label(p, (Bn, 1), (Cn, 1)))] = nijk * R
    elif p.pattern in ("ttv", "ttm") and "_coo3" in p.kernel:
        X = ops["X"]
        On = n["v"] if p.pattern == "ttv" else n["U"]
        nnz = int(X.levels[2].crd.numel())
        if p.kernel == "ttv_coo3_csr":        # gather output: (i, j) then k grouped
            _, nij, nijk = _coo3_level_sizes(X)
            out[(v[0], _label(p, (n["X"], 0)))] = nij
            out[(v[2], _label(p, (n["X"], 2), (On, 0)))] = nijk
        else:                                 # scatter: the fused chain, per nonzero
            out[(v[0], _label(p, (n["X"], 0)))] = nnz
            if p.pattern == "ttm":
                out[(v[3], _label(p, (On, 1)))] = nnz * ops["U"].dims[1]
    elif p.pattern == "plus3":
        out.update(_plus3_counts(p, ops))
    elif p.pattern in ("ttv", "ttm"):
        X = ops["X"]
        On = n["v"] if p.pattern == "ttv" else n["U"]
        nnz = int(X.levels[2].crd.numel())
        out[(v[0], _label(p, (n["X"], 0)))] = int(X.levels[0].crd.numel())
        out[(v[1], _label(p, (n["X"], 1)))] = int(X.levels[1].crd.numel())
        out[(v[2], _label(p, (n["X"], 2), (On, 0)))] = nnz
        if p.pattern == "ttm":
            out[(v[3], _label(p, (On, 1)))] = nnz * ops["U"].dims[1]
    elif p.pattern == "inner":
        out.update(_inner_counts(p, ops))
    return out


def _coo3_level_sizes(X: TensorStorage):
    """Distinct i, (i,j), (i,j,k) of an ordered COO-3 (its grouped levels)."""
    I, J, Kd = X.dims
    i, j, k = (_i64(X.levels[t].crd) for t in range(3))
    if i.numel() == 0:
        return 0, 0, 0
    ij = i * J + j
    return (int(torch.unique_consecutive(i).numel()), int(torch.unique_consecutive(ij).numel()),
            int(torch.unique_consecutive(ij * Kd + k).numel()))


def _spx_visits(pos, crd, xcrd) -> int:
    """Visits of the {A1,x0} intersection loop: per row, the union of the
    row's and x's coordinates up to the smaller of the two last ones."""
    nrows = pos.numel() - 1
    if crd.numel() == 0 or xcrd.numel() == 0:
        return 0
    lens = _i64(pos[1:] - pos[:-1])
    rows = torch.repeat_interleave(torch.arange(nrows, device=pos.device), lens)
    crd = _i64(crd[: rows.numel()])
    xc = _i64(xcrd)
    last_a = torch.where(lens > 0, crd[(_i64(pos[1:]) - 1).clamp(min=0)], torch.full_like(lens, -1))
    m = torch.minimum(last_a, xc[-1].expand_as(last_a))
    live = lens > 0
    in_a = (crd <= m[rows]) & live[rows]
    n_a = torch.zeros(nrows, dtype=torch.int64, device=pos.device).index_add_(0, rows, _i64(in_a))
    shared = torch.zeros(nrows, dtype=torch.int64, device=pos.device).index_add_(
        0, rows, _i64(in_a & torch.isin(crd, xc)))
    n_x = torch.searchsorted(xc, m, right=True)
    return int(torch.where(live, n_a + n_x - shared, torch.zeros_like(n_a)).sum())


def _add_counts(p: Plan, ops, res_csr):
    """Union lattices of C = A + B (lattice.py:346-552): the row loop over
    {A0,B0} then the rows only one side still has; per visited row the column
    loop over {A1,B1}, then {A1} / {B1} for the remainder of the longer row."""
    v = p.ivars
    A, B = ops["A"], ops["B"]
    An, Bn = p.operands["A"], p.operands["B"]
    nrows, ncols = A.dims
    dev = A.vals.device

    def row_keys_and_entries(st):
        if format_class(st.format) == "csr":
            lv, _ = _csr_level(st)
            rows = torch.arange(nrows, dtype=torch.int64, device=dev)   # dense: every row
            return rows, _csr_keys(lv.pos, lv.crd, ncols)
        r, c = st.levels[0].crd, st.levels[1].crd
        rows = torch.unique_consecutive(_i64(r)) if r.numel() else _i64(r)
        return rows, _grouped_keys(r, c, ncols)

    ra, ka = row_keys_and_entries(A)
    rb, kb = row_keys_and_entries(B)
    out = {}
    both_i, a_i, b_i, _ = _merge_counts(ra, rb, max(nrows, 1))
    both_j, a_j, b_j, _ = _merge_counts(ka, kb, ncols)
    out[(v[0], _label(p, (An, 0), (Bn, 0)))] = int(both_i)
    out[(v[0], _label(p, (An, 0)))] = int(a_i)
    out[(v[0], _label(p, (Bn, 0)))] = int(b_i)
    out[(v[1], _label(p, (An, 1), (Bn, 1)))] = int(both_j)
    out[(v[1], _label(p, (An, 1)))] = int(a_j)
    out[(v[1], _label(p, (Bn, 1)))] = int(b_j)
    return out


def _level_keys(st: TensorStorage):
    """Distinct coordinate keys of a COO-3 / CSF operand per level: i,
    i*J + j, (i*J + j)*K + k (sorted)."""
    I, J, Kd = st.dims
    if format_class(st.format) == "coo3":
        i, j, k = (_i64(st.levels[t].crd) for t in range(3))
        if i.numel() == 0:
            return i, i, i
        ij = i * J + j
        return (torch.unique_consecutive(i), torch.unique_consecutive(ij),
                torch.unique_consecutive(ij * Kd + k))
    L = st.levels
    dev = st.vals.device
    s_of_f = torch.repeat_interleave(torch.arange(L[0].crd.numel(), device=dev),
                                     _i64(L[1].pos[1:] - L[1].pos[:-1]))
    fkey = _i64(L[0].crd)[s_of_f] * J + _i64(L[1].crd)
    f_of_l = torch.repeat_interleave(torch.arange(L[1].crd.numel(), device=dev),
                                     _i64(L[2].pos[1:] - L[2].pos[:-1]))
    lkey = fkey[f_of_l] * Kd + _i64(L[2].crd)
    uq = lambda t: torch.unique_consecutive(t) if t.numel() else t  # noqa: E731
    return uq(_i64(L[0].crd)), uq(fkey), uq(lkey)


def _plus3_counts(p: Plan, ops):
    """Union lattices of X + Z at every level (each visited parent's streams
    merged, then the longer one's remainder): (var, {X?,Z?}) visit counts."""
    v = p.ivars
    X, Z = ops["X"], ops["Z"]
    Xn, Zn = p.operands["X"], p.operands["Z"]
    I, J, Kd = X.dims
    kx, kz = _level_keys(X), _level_keys(Z)
    out = {}
    for lvl, (a, b, w) in enumerate(((kx[0], kz[0], 1 << 40), (kx[1], kz[1], J),
                                     (kx[2], kz[2], Kd))):
        both, a_only, b_only, _ = _merge_counts(a, b, w)
        out[(v[lvl], _label(p, (Xn, lvl), (Zn, lvl)))] = int(both)
        out[(v[lvl], _label(p, (Xn, lvl)))] = int(a_only)
        out[(v[lvl], _label(p, (Zn, lvl)))] = int(b_only)
    return out


def _inner_counts(p: Plan, ops):
    """Intersection at every level of two ordered COO-3 tensors: visits of
    each level's merge under the parents matched one level up."""
    v = p.ivars
    X, Z = ops["X"], ops["Z"]
    Xn, Zn = p.operands["X"], p.operands["Z"]
    I, J, Kd = X.dims

    def keys(st):
        i, j, k = (_i64(st.levels[t].crd) for t in range(3))
        if not st.vals.numel() or i.numel() == 0:
            e = i[:0]
            return e, e, e
        ij = i * J + j
        return (torch.unique_consecutive(i), torch.unique_consecutive(ij),
                torch.unique_consecutive(ij * Kd + k))

    (xi, xij, xk), (zi, zij, zk) = keys(X), keys(Z)
    out = {}
    both, _, _, mi = _merge_counts(xi, zi, 1 << 40)     # one root parent
    out[(v[0], _label(p, (Xn, 0), (Zn, 0)))] = int(both)
    keep = lambda k, w, par: k[torch.isin(torch.div(k, w, rounding_mode="floor"), par)]
    xij, zij = keep(xij, J, mi), keep(zij, J, mi)
    both, _, _, mij = _merge_counts(xij, zij, J)
    out[(v[1], _label(p, (Xn, 1), (Zn, 1)))] = int(both)
    xk, zk = keep(xk, Kd, mij), keep(zk, Kd, mij)
    both, _, _, _ = _merge_counts(xk, zk, Kd)
    out[(v[2], _label(p, (Xn, 2), (Zn, 2)))] = int(both)
    return out


_PLAN_CACHE: Dict[tuple, Plan] = {}
_PLAN_CACHE_MAX = 256
_FAST_CACHE: Dict[tuple, tuple] = {}


def _remember(fkey, inputs, out_format, p: Plan) -> None:
    if len(_FAST_CACHE) >= _PLAN_CACHE_MAX:
        _FAST_CACHE.clear()
    _FAST_CACHE[fkey] = (tuple(s.format for s in inputs.values()), out_format, p)


def evaluate(expr, inputs: Dict[str, TensorStorage], out_format: Optional[TensorFormat] = None,
             out_dims: Optional[Sequence[int]] = None, *, fuse: bool = True,
             allow_reorder: bool = True, stats: Optional[EvalStats] = None) -> TensorStorage:
    """Same signature and defaults as the reference (engine.py:739-764).

    Inputs may live on the host (copied to the device first, asynchronously)
    or on a CUDA device; the result is on the device.  `fuse` and
    `allow_reorder` are accepted for signature compatibility: every kernel
    already executes the fused schedule and none needs a reorder stage.
    Plans are cached per (expression text, operand formats and dims, output
    format and dims): parsing, validation and planning are pure functions of
    those, so a repeated call goes straight to the kernels.
    """
    key = None
    if isinstance(expr, str):
        # identity fast path: the same format objects as a cached call skip
        # hashing the (recursive, frozen-dataclass) formats; the entry holds the
        # format objects, so their ids cannot be reused while it is cached
        fkey = (expr, tuple((n, id(s.format), s.dims) for n, s in inputs.items()),
                id(out_format), None if out_dims is None else tuple(out_dims), fuse)
        hit = _FAST_CACHE.get(fkey)
        if hit is not None and all(s.format is f for s, f in zip(inputs.values(), hit[0])) \
                and hit[1] is out_format:
            return _run(hit[2], inputs, stats)
        try:
            key = (expr, tuple(sorted((n, s.format, s.dims) for n, s in inputs.items())),
                   out_format, None if out_dims is None else tuple(out_dims), fuse)
            p = _PLAN_CACHE.get(key)
        except TypeError:            # an unhashable format: plan every time
            key, p = None, None
        if p is not None:
            _remember(fkey, inputs, out_format, p)
            return _run(p, inputs, stats)
    assignment = parse(expr) if isinstance(expr, str) else expr
    bindings = {name: (s.format, s.dims) for name, s in inputs.items()}
    checked = validate(assignment, bindings)
    if out_format is None:
        out_format = preset("dense", order=len(assignment.lhs.ivars))
    if out_dims is None:
        out_dims = tuple(checked.var_extents[v] for v in assignment.lhs.ivars)
    if tuple(out_dims) != tuple(checked.var_extents[v] for v in assignment.lhs.ivars):
        raise ValidationError("out_dims disagree with the expression's variable extents")
    p = plan(checked, bindings, out_format, tuple(out_dims), fuse=fuse)
    if key is not None:
        if len(_PLAN_CACHE) >= _PLAN_CACHE_MAX:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = p
        _remember(fkey, inputs, out_format, p)
    return _run(p, inputs, stats)


def plan_expression(expr, inputs: Dict[str, TensorStorage],
                    out_format: Optional[TensorFormat] = None, *, fuse: bool = True) -> Plan:
    """The kernel binding `evaluate` would use (cf. the reference's `plan`)."""
    assignment = parse(expr) if isinstance(expr, str) else expr
    bindings = {name: (s.format, s.dims) for name, s in inputs.items()}
    checked = validate(assignment, bindings)
    if out_format is None:
        out_format = preset("dense", order=len(assignment.lhs.ivars))
    out_dims = tuple(checked.var_extents[v] for v in assignment.lhs.ivars)
    return plan(checked, bindings, out_format, out_dims, fuse=fuse)
