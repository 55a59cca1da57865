"""Whole-tensor formats composed from levels, and device-resident storage.

TensorFormat / LevelRole / preset mirror the reference's formats.py:33-185
exactly (same presets, aliases and parameters).  TensorStorage holds the level
storages plus a float64 `vals` tensor; arrays live on a CUDA device.  The
`*_storage` constructors wrap arrays already laid out as the reference's
`assemble` lays them out (formats.py:361-501) — the layouts each kernel
consumes; tests/golden/make_golden.py checks the repo's
generators against `assemble` itself.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from .errors import FormatError
from .levels import (LevelKind, LevelSpec, LevelStorage, compressed, dense, hashed, offset_level,
                     range_level, singleton)


@dataclass(frozen=True)
class LevelRole:                                    # formats.py:33-46
    part: str
    mode: int = -1
    factor: int = 1


@dataclass(frozen=True)
class TensorFormat:                                 # formats.py:49-82
    order: int
    levels: Tuple[LevelSpec, ...]
    roles: Tuple[LevelRole, ...]
    mode_ordering: Tuple[int, ...]
    name: str = ""
    aos: bool = False
    hash_width: int = 0
    params: Tuple[Tuple[str, int], ...] = ()

    def __post_init__(self):
        if len(self.levels) != len(self.roles):
            raise FormatError("levels and roles must align")
        if sorted(self.mode_ordering) != list(range(self.order)):
            raise FormatError(f"mode ordering {self.mode_ordering} is not a permutation")
        for spec in self.levels:
            if not (spec.value_iterable or spec.position_iterable):
                raise FormatError("every level must support value or position iteration")

    @property
    def structured(self) -> bool:
        return any(r.part != "whole" for r in self.roles)

    def param(self, key: str, default: int = 0) -> int:
        return dict(self.params).get(key, default)

    def describe(self) -> str:
        body = ",".join(spec.describe() for spec in self.levels)
        suffix = ""
        if self.mode_ordering != tuple(range(self.order)):
            suffix = "@(" + ",".join(map(str, self.mode_ordering)) + ")"
        return "{" + body + "}" + suffix

    def kinds(self) -> Tuple[LevelKind, ...]:
        return tuple(s.kind for s in self.levels)


def _whole_roles(mode_ordering):
    return tuple(LevelRole("whole", m) for m in mode_ordering)


def simple_format(levels: Sequence[LevelSpec], mode_ordering: Optional[Sequence[int]] = None,
                  name: str = "", aos: bool = False, hash_width: int = 0) -> TensorFormat:
    order = len(levels)
    mo = tuple(mode_ordering) if mode_ordering is not None else tuple(range(order))
    return TensorFormat(order, tuple(levels), _whole_roles(mo), mo, name=name, aos=aos,
                        hash_width=hash_width)


_PRESET_ALIASES = {                                 # formats.py:98-102
    "coo": "coo-soa", "coo-2": "coo-soa", "coo3": "coo-3", "coo-3-soa": "coo-3",
    "sv": "sparse-vector", "hash": "hash-vector", "mg": "mode-generic",
    "dense-1": "dense", "dense1": "dense",
}


def preset(name: str, order: Optional[int] = None, *, block: int = 2, slots: int = 0,
           width: int = 0, inner: int = 1) -> TensorFormat:
    """The stock formats of formats.py:105-185 (Fig. 5 of the paper)."""
    key = _PRESET_ALIASES.get(name.strip().lower(), name.strip().lower())
    if key == "dense":
        n = order if order is not None else 1
        return simple_format([dense() for _ in range(n)], name="dense")
    if key == "dense-2":
        return simple_format([dense(), dense()], name="dense")
    if key == "dense-3":
        return simple_format([dense(), dense(), dense()], name="dense")
    if key == "sparse-vector":
        return simple_format([compressed()], name="sparse-vector")
    if key == "hash-vector":
        return simple_format([hashed()], name="hash-vector", hash_width=width)
    if key == "csr":
        return simple_format([dense(), compressed()], name="csr")
    if key == "csc":
        return simple_format([dense(), compressed()], mode_ordering=(1, 0), name="csc")
    if key == "dcsr":
        return simple_format([compressed(), compressed()], name="dcsr")
    if key == "coo-soa":
        return simple_format([compressed(unique=False), singleton()], name="coo-soa")
    if key == "coo-aos":
        return simple_format([compressed(unique=False), singleton()], name="coo-aos", aos=True)
    if key == "csf":
        return simple_format([compressed(), compressed(), compressed()], name="csf")
    if key == "coo-3":
        return simple_format([compressed(unique=False), singleton(unique=False), singleton()],
                             name="coo-3")
    if key == "coo-3-aos":
        return simple_format([compressed(unique=False), singleton(unique=False), singleton()],
                             name="coo-3-aos", aos=True)
    if key == "bcsr":
        if block < 1:
            raise FormatError("BCSR block size must be positive")
        return TensorFormat(2, (dense(), compressed(), dense(), dense()),
                            (LevelRole("block", 0, block), LevelRole("block", 1, block),
                             LevelRole("inner", 0, block), LevelRole("inner", 1, block)),
                            (0, 1), name="bcsr", params=(("block", block),))
    if key == "csb":
        if block < 1:
            raise FormatError("CSB block size must be positive")
        return TensorFormat(2, (dense(), dense(), compressed(ordered=False, unique=False),
                                singleton(ordered=False)),
                            (LevelRole("block", 0, block), LevelRole("block", 1, block),
                             LevelRole("inner", 0, block), LevelRole("inner", 1, block)),
                            (0, 1), name="csb", params=(("block", block),))
    if key == "ell":
        return TensorFormat(2, (dense(), dense(), singleton()),
                            (LevelRole("slot"), LevelRole("whole", 0), LevelRole("whole", 1)),
                            (0, 1), name="ell", params=(("slots", slots),))
    if key == "dia":
        return TensorFormat(2, (dense(), range_level(), offset_level()),
                            (LevelRole("diag"), LevelRole("whole", 0), LevelRole("whole", 1)),
                            (0, 1), name="dia")
    if key == "mode-generic":
        if inner < 1:
            raise FormatError("mode-generic inner block size must be positive")
        return TensorFormat(3, (compressed(unique=False), singleton(), dense(), dense()),
                            (LevelRole("whole", 0), LevelRole("block", 1, inner),
                             LevelRole("inner", 1, inner), LevelRole("whole", 2)),
                            (0, 1, 2), name="mode-generic", params=(("inner", inner),))
    raise FormatError(f"unknown format preset: {name!r}")


PRESET_NAMES = ["dense", "sparse-vector", "hash-vector", "csr", "csc", "dcsr", "coo-soa",
                "coo-aos", "bcsr", "ell", "dia", "csb", "csf", "coo-3", "mode-generic"]


class TensorStorage:
    """A tensor format instantiated with level storages and a values tensor
    (formats.py:244-263).  `vals` is a float64 tensor on the same device."""

    def __init__(self, fmt: TensorFormat, dims, levels, vals):
        self.format = fmt
        self.dims = tuple(int(d) for d in dims)
        self.levels = list(levels)
        self.vals = vals

    @property
    def order(self) -> int:
        return self.format.order

    @property
    def device(self):
        return self.vals.device

    def to(self, device, non_blocking: bool = False) -> "TensorStorage":
        import torch

        lv = [level.to(device) for level in self.levels]
        vals = self.vals.to(device=device, dtype=torch.float64, non_blocking=non_blocking)
        return TensorStorage(self.format, self.dims, lv, vals)

    def __repr__(self):
        return (f"TensorStorage({self.format.name or self.format.describe()}, dims={self.dims}, "
                f"vals={int(self.vals.numel())}, device={self.vals.device})")


# ---------------------------------------------------------------------------
# constructors over arrays in assemble() layout

def _f64(a, device, pin=False):
    import torch

    if isinstance(a, torch.Tensor):
        t = a.to(dtype=torch.float64)
        return t.to(device) if device is not None else t
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64))
    if pin and device is None:
        t = t.pin_memory()
    return t.to(device) if device is not None else t


def dense_storage(values, dims=None, device="cuda") -> TensorStorage:
    """Dense vector/matrix/3-tensor, row-major (dense-N preset)."""
    vals = _f64(values, device)
    dims = tuple(dims) if dims is not None else tuple(vals.shape) or (1,)
    fmt = preset("dense", len(dims))
    levels = [LevelStorage(spec, n=n, device=vals.device) for spec, n in zip(fmt.levels, dims)]
    return TensorStorage(fmt, dims, levels, vals.reshape(-1))


def coo_storage(rows, cols, vals, dims, device="cuda") -> TensorStorage:
    """COO-SoA (formats.py:132-133): L0 compressed(~U) pos=[0,nnz] crd=rows,
    L1 singleton crd=cols; row-major sorted."""
    fmt = preset("coo-soa")
    nnz = len(rows)
    l0 = LevelStorage(fmt.levels[0], pos=[0, nnz], crd=rows, device=device)
    l1 = LevelStorage(fmt.levels[1], crd=cols, device=device)
    return TensorStorage(fmt, dims, [l0, l1], _f64(vals, device))


def csr_storage(pos, crd, vals, dims, device="cuda") -> TensorStorage:
    """CSR (formats.py:126-127): dense rows + compressed columns."""
    fmt = preset("csr")
    l0 = LevelStorage(fmt.levels[0], n=dims[0], device=device)
    l1 = LevelStorage(fmt.levels[1], pos=pos, crd=crd, device=device)
    return TensorStorage(fmt, dims, [l0, l1], _f64(vals, device))


def ell_storage(nslots, crd, vals, dims, device="cuda") -> TensorStorage:
    """ELL (formats.py:164-169): dense(slots) + dense(rows) + singleton,
    slot-major positions s*N + i, padding (col 0, 0.0)."""
    fmt = preset("ell", slots=nslots)
    l0 = LevelStorage(fmt.levels[0], n=nslots, device=device)
    l1 = LevelStorage(fmt.levels[1], n=dims[0], device=device)
    l2 = LevelStorage(fmt.levels[2], crd=crd, device=device)
    return TensorStorage(fmt, dims, [l0, l1, l2], _f64(vals, device))


def dia_storage(offsets, vals, dims, device="cuda") -> TensorStorage:
    """DIA (formats.py:170-175): dense(diagonals) + range + offset sharing one
    sorted offset array; vals at d*N + i."""
    fmt = preset("dia")
    offs = np.asarray(offsets, dtype=np.int32)
    if len(offs) > 1 and not (np.diff(offs) > 0).all():
        raise FormatError("DIA offsets must be sorted ascending and distinct")
    l0 = LevelStorage(fmt.levels[0], n=len(offs), device=device)
    l1 = LevelStorage(fmt.levels[1], n=dims[0], m=dims[1], offset=offs, device=device)
    l2 = LevelStorage(fmt.levels[2], offset=l1.offset, range_n=dims[0], device=device)
    l2.offset = l1.offset  # shared array, as in the reference (formats.py:394, 405-412)
    st = TensorStorage(fmt, dims, [l0, l1, l2], _f64(vals, device))
    st._host_offsets = offs.copy()
    return st


def sparse_vector_storage(crd, vals, n, device="cuda") -> TensorStorage:
    """sparse-vector (formats.py:122-123): one compressed level, sorted unique
    coordinates, pos = [0, nnz]."""
    fmt = preset("sparse-vector")
    crd = np.asarray(crd, dtype=np.int32) if not hasattr(crd, "is_cuda") else crd
    nnz = len(crd)
    l0 = LevelStorage(fmt.levels[0], pos=[0, nnz], crd=crd, device=device)
    return TensorStorage(fmt, (n,), [l0], _f64(vals, device))


def hash_vector_storage(crd, vals, n, width, device="cuda") -> TensorStorage:
    """hash-vector (formats.py:124-125): one hashed level of width W,
    crd[W] with -1 empties, vals[W] by slot."""
    fmt = preset("hash-vector", width=width)
    l0 = LevelStorage(fmt.levels[0], w=width, crd=crd, device=device)
    return TensorStorage(fmt, (n,), [l0], _f64(vals, device))


def coo3_storage(i, j, k, vals, dims, device="cuda") -> TensorStorage:
    """COO-3 (formats.py:138-140): compressed(~U) + singleton(~U) + singleton."""
    fmt = preset("coo-3")
    nnz = len(i)
    l0 = LevelStorage(fmt.levels[0], pos=[0, nnz], crd=i, device=device)
    l1 = LevelStorage(fmt.levels[1], crd=j, device=device)
    l2 = LevelStorage(fmt.levels[2], crd=k, device=device)
    return TensorStorage(fmt, dims, [l0, l1, l2], _f64(vals, device))


def csf_storage(pos0, crd0, pos1, crd1, pos2, crd2, vals, dims, device="cuda") -> TensorStorage:
    """CSF (formats.py:136-137): three compressed levels."""
    fmt = preset("csf")
    lv = [LevelStorage(fmt.levels[0], pos=pos0, crd=crd0, device=device),
          LevelStorage(fmt.levels[1], pos=pos1, crd=crd1, device=device),
          LevelStorage(fmt.levels[2], pos=pos2, crd=crd2, device=device)]
    return TensorStorage(fmt, dims, lv, _f64(vals, device))


# ---------------------------------------------------------------------------
# conversion

def convert(src: TensorStorage, dst: TensorFormat) -> TensorStorage:
    """Re-store `src` in format `dst` (formats.py:583-587: an identity
    assignment `OUT(i,j) = IN(i,j)` evaluated by the engine, engine.py:775-779).

    Device kernels (csrc/convert.cu, csrc/add.cu) reproduce the reference's
    output exactly:
      COO -> CSR : gather-append copy — duplicates summed +0.0 + v1 + ...,
                   stored 0.0 + value, explicit zeros kept (A+B kernels, A empty)
      CSR -> ELL : reorder writer + assemble — exact zeros dropped, 0.0 + v
      COO -> ELL : COO -> CSR -> ELL (same values as the direct copy)
      COO -> DIA : reorder writer + assemble (unique coordinates)
      CSR -> COO : gather-append copy (0.0 + v, explicit zeros kept)
    Other pairs raise UnsupportedOutputError (no CPU interpretation)."""
    from . import kernels as K
    from .engine import format_class
    from .errors import UnsupportedOutputError

    s, d = format_class(src.format), format_class(dst)
    dims = tuple(src.dims)
    if len(dims) != 2:
        raise UnsupportedOutputError(f"no device conversion {s} -> {d}")
    n, m = dims
    dev = src.vals.device
    if s == "coo" and d in ("csr", "ell"):
        pos, crd, vals = K.coo_to_csr(n, src.levels[0].crd, src.levels[1].crd, src.vals)
        csr = csr_storage(pos, crd, vals, dims, device=dev)
        return csr if d == "csr" else convert(csr, dst)
    if s == "csr" and d == "ell":
        l1 = src.levels[1]
        nslots, ecrd, evals = K.csr_to_ell(n, l1.pos, l1.crd, src.vals)
        return ell_storage(nslots, ecrd, evals, dims, device=dev)
    if s == "csr" and d == "coo":
        l1 = src.levels[1]
        rows, cols, vals = K.csr_to_coo(n, l1.pos, l1.crd, src.vals)
        return coo_storage(rows, cols, vals, dims, device=dev)
    if s == "coo" and d == "dia":
        offs, dvals = K.coo_to_dia(n, m, src.levels[0].crd, src.levels[1].crd, src.vals)
        return dia_storage(offs.cpu().numpy(), dvals, dims, device=dev)
    raise UnsupportedOutputError(f"no device conversion {s} -> {d}")
