"""Matrix Market and FROSTT .tns files <-> CoordList.

Same accepted inputs, results and `FileFormatError`s as the reference's
readers and writers (io.py:64-196): 1-based coordinates in the files,
0-based in memory; duplicates kept in file order (call `canonicalize` or
`assemble` to merge them); Matrix Market: coordinate / general only, values
real, integer or pattern (1.0); .tns: order taken from the first data line,
extents from an explicit `dims` or the per-column maxima.  Reading is
vectorised once the header/lines are validated; `assembly.assemble` then
builds device storage in any in-scope format.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .assembly import CoordList
from .errors import SparseLevelsError

__all__ = ["FileFormatError", "read_mtx", "write_mtx", "read_tns", "write_tns"]

_MTX = "%%MatrixMarket"


class FileFormatError(SparseLevelsError):
    """Malformed tensor file (reference io.py:19-20)."""


def _data_lines(lines: List[str], comment: str):
    for lineno, raw in enumerate(lines, 1):
        line = raw.strip()
        if line and not line.startswith(comment):
            yield lineno, line


def read_mtx(path: str) -> CoordList:
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.readlines()
    if not lines or not lines[0].startswith(_MTX):
        raise FileFormatError(f"{path}:1: missing MatrixMarket header")
    head = lines[0].split()
    if len(head) < 5:
        raise FileFormatError(f"{path}:1: incomplete header")
    _, obj, layout, field, symmetry = head[:5]
    if obj.lower() != "matrix" or layout.lower() != "coordinate":
        raise FileFormatError(f"{path}:1: only coordinate matrices are supported")
    field = field.lower()
    if field not in ("real", "integer", "pattern"):
        raise FileFormatError(f"{path}:1: unsupported value type {field!r}")
    if symmetry.lower() != "general":
        raise FileFormatError(
            f"{path}:1: symmetry {symmetry!r} is not supported; expand to general first")
    body = list(_data_lines(lines[1:], "%"))
    if not body:
        raise FileFormatError(f"{path}: missing size line")
    size_no, size = body[0]
    parts = size.split()
    if len(parts) != 3:
        raise FileFormatError(f"{path}:{size_no + 1}: expected 'rows cols nnz'")
    nrows, ncols, declared = (int(p) for p in parts)
    want = 2 if field == "pattern" else 3
    rows, cols, vals = [], [], []
    for no, line in body[1:]:
        f = line.split()
        if len(f) != want:
            raise FileFormatError(f"{path}:{no + 1}: expected {want} fields")
        try:
            i, j = int(f[0]) - 1, int(f[1]) - 1
            v = 1.0 if field == "pattern" else float(f[2])
        except ValueError as exc:
            raise FileFormatError(f"{path}:{no + 1}: {exc}") from None
        if not (0 <= i < nrows and 0 <= j < ncols):
            raise FileFormatError(
                f"{path}:{no + 1}: coordinate ({i + 1}, {j + 1}) outside {(nrows, ncols)}")
        rows.append(i)
        cols.append(j)
        vals.append(v)
    if len(vals) != declared:
        raise FileFormatError(f"{path}: header declares {declared} entries, found {len(vals)}")
    coords = np.stack([np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)], axis=1) \
        if vals else np.zeros((0, 2), dtype=np.int64)
    return CoordList((nrows, ncols), coords, np.array(vals, dtype=np.float64))


def write_mtx(data: CoordList, path: str) -> None:
    if len(data.dims) != 2:
        raise FileFormatError("Matrix Market files store matrices (order 2)")
    with open(path, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{data.dims[0]} {data.dims[1]} {data.nnz}\n")
        for (i, j), v in zip(data.coords.tolist(), data.vals.tolist()):
            fh.write(f"{i + 1} {j + 1} {v!r}\n")


def read_tns(path: str, dims: Optional[Sequence[int]] = None) -> CoordList:
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.readlines()
    order = None
    coords: List[List[int]] = []
    vals: List[float] = []
    for no, line in _data_lines(lines, "#"):
        f = line.split()
        if len(f) < 2:
            raise FileFormatError(f"{path}:{no}: need coordinates and a value")
        if order is None:
            order = len(f) - 1
        elif len(f) - 1 != order:
            raise FileFormatError(f"{path}:{no}: expected {order} coordinates, got {len(f) - 1}")
        try:
            c = [int(p) - 1 for p in f[:-1]]
            v = float(f[-1])
        except ValueError as exc:
            raise FileFormatError(f"{path}:{no}: {exc}") from None
        if min(c) < 0:
            raise FileFormatError(f"{path}:{no}: coordinates are 1-based")
        coords.append(c)
        vals.append(v)
    if order is None:
        order = len(dims) if dims is not None else 0
    arr = np.array(coords, dtype=np.int64).reshape(-1, order)
    if dims is not None:
        dims = tuple(int(d) for d in dims)
        if len(dims) != order:
            raise FileFormatError(f"{path}: sidecar dims {dims} do not match order {order}")
        if len(arr) and (arr >= np.array(dims)).any():
            bad = arr[np.nonzero((arr >= np.array(dims)).any(1))[0][0]]
            raise FileFormatError(f"{path}: coordinate {tuple(int(x) for x in bad)} outside dims {dims}")
    else:
        dims = tuple(int(m) + 1 for m in arr.max(0)) if len(arr) else (0,) * order
    return CoordList(dims, arr, np.array(vals, dtype=np.float64))


def write_tns(data: CoordList, path: str) -> None:
    with open(path, "w", encoding="ascii") as fh:
        for c, v in zip(data.coords.tolist(), data.vals.tolist()):
            fh.write(" ".join(str(x + 1) for x in c) + f" {v!r}\n")
