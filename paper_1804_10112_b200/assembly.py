"""Coordinate lists -> storage in every in-scope format (host side of the
boundary: the data formats on either side of the hot path).

Mirrors the reference's `CoordList`, `canonicalize` and `assemble`
(formats.py:195-222, 361-501) with the same results, vectorised in numpy:

* formats whose levels are all unique canonicalise first: duplicates summed in
  input order from +0.0 (0.0 + v1 + v2 ...), entries sorted, exact zeros
  dropped (formats.py:217-222);
* formats with a non-unique level (COO-SoA, COO-3) keep every entry, stably
  sorted into storage order (formats.py:376-388);
* every stored value is 0.0 + value (formats.py:498-500: vals[pos] += value),
  so -0.0 is stored as +0.0.

The result is a device `TensorStorage` built by the `*_storage` constructors.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence, Tuple, Union

import numpy as np

from .errors import AssemblyError
from .formats import (TensorFormat, TensorStorage, coo3_storage, coo_storage, csf_storage,
                      csr_storage, dense_storage, dia_storage, ell_storage, hash_vector_storage,
                      preset, sparse_vector_storage)


@dataclass
class CoordList:
    """Coordinates (nnz x order, int64) and values (float64) of a tensor
    (formats.py:195-214).  `canonical` = unique, sorted, no explicit zeros."""

    dims: Tuple[int, ...]
    coords: np.ndarray
    vals: np.ndarray
    canonical: bool = False

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        self.coords = np.asarray(self.coords, dtype=np.int64).reshape(-1, len(self.dims))
        self.vals = np.asarray(self.vals, dtype=np.float64).reshape(-1)
        if len(self.vals) != len(self.coords):
            raise AssemblyError(f"{len(self.coords)} coordinates but {len(self.vals)} values")

    @classmethod
    def from_entries(cls, dims, entries, canonical=False) -> "CoordList":
        """From the reference's [((c0, c1, ...), value), ...] form."""
        order = len(tuple(dims))
        coords = np.array([c for c, _ in entries], dtype=np.int64).reshape(-1, order)
        vals = np.array([v for _, v in entries], dtype=np.float64)
        return cls(dims, coords, vals, canonical)

    @property
    def nnz(self) -> int:
        return len(self.vals)


def _check_bounds(data: CoordList) -> None:
    if data.nnz and ((data.coords < 0).any() or (data.coords >= np.array(data.dims)).any()):
        bad = np.nonzero(((data.coords < 0) | (data.coords >= np.array(data.dims))).any(1))[0][0]
        raise AssemblyError(f"coordinate {tuple(int(c) for c in data.coords[bad])} "
                            f"outside dims {data.dims}")


def _lex_order(coords: np.ndarray) -> np.ndarray:
    """Stable lexicographic order of the rows of `coords`."""
    if coords.shape[0] == 0:
        return np.zeros(0, dtype=np.int64)
    return np.lexsort(tuple(coords[:, k] for k in range(coords.shape[1] - 1, -1, -1)))


def canonicalize(data: CoordList) -> CoordList:
    """formats.py:217-222: sum duplicates in input order from +0.0, sort,
    drop exact zeros."""
    if data.nnz == 0:
        return CoordList(data.dims, data.coords, data.vals, True)
    order = _lex_order(data.coords)
    c, v = data.coords[order], data.vals[order]
    new = np.ones(len(v), dtype=bool)
    new[1:] = (c[1:] != c[:-1]).any(1)
    starts = np.nonzero(new)[0]
    sums = 0.0 + v[starts]
    ends = np.append(starts[1:], len(v))
    for g in np.nonzero(ends - starts > 1)[0]:          # duplicate groups, in input order
        acc = 0.0
        for t in v[starts[g]:ends[g]]:
            acc = acc + float(t)
        sums[g] = acc
    keep = sums != 0.0
    return CoordList(data.dims, c[starts][keep], sums[keep], True)


def _unique_format(fmt: TensorFormat) -> bool:
    return all(spec.props.unique for spec in fmt.levels)


def assemble(fmt: Union[str, TensorFormat], dims: Sequence[int], data: CoordList,
             diagonals: Optional[Sequence[int]] = None, device="cuda") -> TensorStorage:
    """Build device storage for `data` (formats.py:361-501).  Formats:
    dense-N, sparse-vector, hash-vector, CSR, COO-SoA, ELL, DIA, COO-3, CSF."""
    from .engine import format_class

    fmt = preset(fmt) if isinstance(fmt, str) else fmt
    dims = tuple(int(d) for d in dims)
    if len(dims) != fmt.order:
        raise AssemblyError(f"dims {dims} do not match format order {fmt.order}")
    if data.dims != dims:
        data = CoordList(dims, data.coords, data.vals, data.canonical)
    _check_bounds(data)
    if _unique_format(fmt) and not data.canonical:
        data = canonicalize(data)
    cls = format_class(fmt)
    order = _lex_order(data.coords)                      # storage order (stable)
    c, v = data.coords[order], 0.0 + data.vals[order]
    n = len(v)
    if cls.startswith("dense"):
        if not dims:                                     # a scalar
            from .formats import _f64
            val = np.array([0.0 + float(v.sum()) if n else 0.0])
            return TensorStorage(fmt, (), [], _f64(val, device))
        flat = np.zeros(int(np.prod(dims)))
        if n:
            flat[np.ravel_multi_index(tuple(c[:, k] for k in range(len(dims))), dims)] = v
        return dense_storage(flat.reshape(dims), dims, device=device)
    if cls == "spvec":
        return sparse_vector_storage(c[:, 0].astype(np.int32), v, dims[0], device=device)
    if cls == "hash1":
        from .workloads import hash_insert_sequential
        w = fmt.hash_width
        if not w:                                        # _next_pow2(max(4, 2 * extent))
            w = 1
            while w < max(4, 2 * dims[0]):
                w *= 2
        crd, slots = hash_insert_sequential(c[:, 0], w)
        vals = np.zeros(w)
        vals[slots] = v
        return hash_vector_storage(crd, vals, dims[0], w, device=device)
    if cls == "coo":
        return coo_storage(c[:, 0].astype(np.int32), c[:, 1].astype(np.int32), v, dims,
                           device=device)
    if cls == "coo3":
        return coo3_storage(c[:, 0].astype(np.int32), c[:, 1].astype(np.int32),
                            c[:, 2].astype(np.int32), v, dims, device=device)
    if cls == "csr":
        pos = np.zeros(dims[0] + 1, dtype=np.int64)
        np.cumsum(np.bincount(c[:, 0], minlength=dims[0]), out=pos[1:])
        return csr_storage(pos.astype(np.int32), c[:, 1].astype(np.int32), v, dims, device=device)
    if cls == "ell":
        N = dims[0]
        counts = np.bincount(c[:, 0], minlength=N)
        S = int(counts.max()) if n else 0
        declared = fmt.param("slots", 0)
        if declared:
            if S > declared:
                raise AssemblyError(f"row with {S} entries exceeds the declared slot count "
                                    f"{declared}")
            S = declared
        start = np.zeros(N + 1, dtype=np.int64)
        np.cumsum(counts, out=start[1:])
        slot = np.arange(n) - start[c[:, 0]]
        crd = np.zeros(S * N, dtype=np.int32)
        vals = np.zeros(S * N)
        crd[slot * N + c[:, 0]] = c[:, 1]
        vals[slot * N + c[:, 0]] = v
        return ell_storage(S, crd, vals, dims, device=device)
    if cls == "dia":
        N = dims[0]
        d = c[:, 1] - c[:, 0]
        offs = np.unique(d)
        if diagonals is not None:
            declared = np.unique(np.asarray(diagonals, dtype=np.int64))
            extra = np.setdiff1d(offs, declared)
            if len(extra):
                raise AssemblyError(f"data has diagonals {extra.tolist()} not in the declared "
                                    f"set {declared.tolist()}")
            offs = declared
        di = np.searchsorted(offs, d)
        vals = np.zeros(len(offs) * N)
        vals[di * N + c[:, 0]] = v
        return dia_storage(offs.astype(np.int32), vals, dims, device=device)
    if cls == "csf":
        new_i = np.ones(n, dtype=bool)
        new_i[1:] = c[1:, 0] != c[:-1, 0]
        new_f = new_i.copy()
        new_f[1:] |= c[1:, 1] != c[:-1, 1]
        si = np.nonzero(new_i)[0]
        fi = np.nonzero(new_f)[0]
        pos1 = np.searchsorted(fi, si).tolist() + [len(fi)]
        pos2 = fi.tolist() + [n]
        return csf_storage(np.array([0, len(si)], np.int32), c[si, 0].astype(np.int32),
                           np.array(pos1, np.int32), c[fi, 1].astype(np.int32),
                           np.array(pos2, np.int32), c[:, 2].astype(np.int32), v, dims,
                           device=device)
    raise AssemblyError(f"no assembly for format {fmt.describe()} (in-scope: dense, "
                        "sparse-vector, hash-vector, CSR, COO-SoA, ELL, DIA, COO-3, CSF)")
