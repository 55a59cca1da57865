"""Per-dimension level formats and the level-function interface (device-backed).

Same names, capability sets, property model and error behaviour as the
reference's levels.py.  The difference is where the arrays live and who runs
the level functions: LevelStorage holds CUDA tensors, and its access
functions execute the inlined device level functions of csrc/levels.cuh
through the batched C-ABI entry `sl_level_query` (scalar calls are a batch
of one).  Capability violations raise UnsupportedCapabilityError before any
launch, as LevelStorage._require does (levels.py:197-199).
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass
from typing import Sequence, Tuple

from . import _lib
from .errors import (AssemblyError, FormatError, HashSegmentFullError,
                     UnsupportedCapabilityError)


class LevelKind(enum.Enum):                       # levels.py:25-31
    DENSE = "dense"
    RANGE = "range"
    COMPRESSED = "compressed"
    SINGLETON = "singleton"
    OFFSET = "offset"
    HASHED = "hashed"


# Access and assembly capabilities per kind (levels.py:35-41).
VALUE_ITERATION = frozenset({LevelKind.DENSE, LevelKind.RANGE})
POSITION_ITERATION = frozenset(
    {LevelKind.COMPRESSED, LevelKind.SINGLETON, LevelKind.OFFSET, LevelKind.HASHED})
LOCATE_CAPABLE = frozenset({LevelKind.DENSE, LevelKind.HASHED})
INSERT_CAPABLE = frozenset({LevelKind.DENSE, LevelKind.HASHED})
APPEND_CAPABLE = frozenset({LevelKind.COMPRESSED, LevelKind.SINGLETON})

EMPTY = -1  # levels.py:43


@dataclass(frozen=True)
class PropertySet:                                 # levels.py:46-54
    full: bool
    ordered: bool
    unique: bool
    branchless: bool
    compact: bool


# Per kind: fixed property values; None = configurable (levels.py:57-65).
_FIXED = {
    LevelKind.DENSE: dict(full=True, ordered=None, unique=None, branchless=False, compact=True),
    LevelKind.RANGE: dict(full=False, ordered=None, unique=None, branchless=False, compact=False),
    LevelKind.COMPRESSED: dict(full=None, ordered=None, unique=None, branchless=False,
                               compact=True),
    LevelKind.SINGLETON: dict(full=None, ordered=None, unique=None, branchless=True,
                              compact=True),
    LevelKind.OFFSET: dict(full=False, ordered=None, unique=None, branchless=True, compact=False),
    LevelKind.HASHED: dict(full=None, ordered=False, unique=None, branchless=False,
                           compact=False),
}
_DEFAULTS = dict(full=False, ordered=True, unique=True)   # levels.py:68
_NAMES = ("full", "ordered", "unique", "branchless", "compact")


def make_properties(kind: LevelKind, **flags) -> PropertySet:
    """levels.py:71-93: configurable flags default to full=False,
    ordered=True, unique=True; contradicting a fixed flag is a FormatError."""
    fixed = _FIXED[kind]
    values = {}
    for name in _NAMES:
        want = flags.pop(name, None)
        allowed = fixed[name]
        if allowed is None:
            values[name] = _DEFAULTS[name] if want is None else bool(want)
        else:
            if want is not None and bool(want) != allowed:
                raise FormatError(
                    f"{kind.value} level is always {name}={allowed}; cannot set {name}={want}")
            values[name] = allowed
    if flags:
        raise FormatError(f"unknown property flags: {sorted(flags)}")
    return PropertySet(**values)


@dataclass(frozen=True)
class LevelSpec:                                   # levels.py:96-130
    kind: LevelKind
    props: PropertySet

    @property
    def value_iterable(self) -> bool:
        return self.kind in VALUE_ITERATION

    @property
    def position_iterable(self) -> bool:
        return self.kind in POSITION_ITERATION

    @property
    def locate_capable(self) -> bool:
        return self.kind in LOCATE_CAPABLE

    @property
    def insert_capable(self) -> bool:
        return self.kind in INSERT_CAPABLE

    @property
    def append_capable(self) -> bool:
        return self.kind in APPEND_CAPABLE

    def describe(self) -> str:
        tags = []
        for name, short in (("full", "f"), ("ordered", "o"), ("unique", "u")):
            default = _DEFAULTS[name] if _FIXED[self.kind][name] is None else _FIXED[self.kind][name]
            actual = getattr(self.props, name)
            if actual != default:
                tags.append(short if actual else "~" + short)
        return self.kind.value + (f"({','.join(tags)})" if tags else "")


def dense(**flags) -> LevelSpec:
    return LevelSpec(LevelKind.DENSE, make_properties(LevelKind.DENSE, **flags))


def range_level(**flags) -> LevelSpec:
    return LevelSpec(LevelKind.RANGE, make_properties(LevelKind.RANGE, **flags))


def compressed(**flags) -> LevelSpec:
    return LevelSpec(LevelKind.COMPRESSED, make_properties(LevelKind.COMPRESSED, **flags))


def singleton(**flags) -> LevelSpec:
    return LevelSpec(LevelKind.SINGLETON, make_properties(LevelKind.SINGLETON, **flags))


def offset_level(**flags) -> LevelSpec:
    return LevelSpec(LevelKind.OFFSET, make_properties(LevelKind.OFFSET, **flags))


def hashed(**flags) -> LevelSpec:
    return LevelSpec(LevelKind.HASHED, make_properties(LevelKind.HASHED, **flags))


def _as_i32(a, device):
    import numpy as np
    import torch

    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=device)


class LevelStorage:
    """Physical storage of one coordinate-hierarchy level (levels.py:157-191).

    Fields are the reference's: spec, n, m, w, pos, crd, offset, crd_stride,
    crd_base, range_n.  Array fields are int32 CUDA tensors (numpy or lists
    are moved to `device` on construction).  Storage is immutable after
    assembly; concurrent reads are safe.
    """

    __slots__ = ("spec", "n", "m", "w", "pos", "crd", "offset", "crd_stride", "crd_base",
                 "range_n", "_appended", "_edges", "_last_edge_parent", "_sl_max_row")

    def __init__(self, spec: LevelSpec, *, n: int = 0, m: int = 0, w: int = 0, pos=None, crd=None,
                 offset=None, crd_stride: int = 1, crd_base: int = 0, range_n: int = 0,
                 device="cuda"):
        self.spec = spec
        self._sl_max_row = None   # (pos, heaviest 32-row tile): engine's CSR variant choice, cached
        self.n, self.m, self.w = int(n), int(m), int(w)
        # the reference defaults pos / crd to [] (levels.py:185-186): position
        # iterated levels always carry (possibly empty) arrays here too
        if spec.kind in (LevelKind.COMPRESSED, LevelKind.SINGLETON, LevelKind.HASHED):
            crd = [] if crd is None else crd
            if spec.kind is LevelKind.COMPRESSED:
                pos = [] if pos is None else pos
        self.pos = _as_i32(pos, device)
        self.crd = _as_i32(crd, device)
        self.offset = _as_i32(offset, device)
        self.crd_stride, self.crd_base, self.range_n = int(crd_stride), int(crd_base), int(range_n)
        self._appended = None
        self._edges = None
        self._last_edge_parent = -1

    @property
    def kind(self) -> LevelKind:
        return self.spec.kind

    def to(self, device) -> "LevelStorage":
        out = LevelStorage(self.spec, n=self.n, m=self.m, w=self.w, crd_stride=self.crd_stride,
                           crd_base=self.crd_base, range_n=self.range_n, device=device)
        out.pos = None if self.pos is None else self.pos.to(device)
        out.crd = None if self.crd is None else self.crd.to(device)
        out.offset = None if self.offset is None else self.offset.to(device)
        return out

    def _require(self, capability: frozenset, fn: str) -> None:
        if self.kind not in capability:
            raise UnsupportedCapabilityError(f"{self.kind.value} level does not support {fn}")

    # -- device descriptor --------------------------------------------------

    def descriptor(self) -> _lib.SlLevel:
        d = _lib.SlLevel()
        d.kind = _lib.KIND_ID[self.kind.value]
        d.crd_stride, d.crd_base = self.crd_stride, self.crd_base
        d.noffset = 0 if self.offset is None else int(self.offset.numel())
        d.n, d.m, d.w, d.range_n = self.n, self.m, self.w, self.range_n
        d.pos = _lib.ptr(self.pos)
        d.crd = _lib.ptr(self.crd)
        d.offset = _lib.ptr(self.offset)
        return d

    def query(self, fn: str, a, b=None):
        """Batched level function on the device: returns (o0, o1) int64 CUDA
        tensors.  `fn` is one of coord_bounds, coord_access, pos_bounds,
        pos_access, locate, size (levels.py:215-294)."""
        import torch

        cap = {"coord_bounds": VALUE_ITERATION, "coord_access": VALUE_ITERATION,
               "pos_bounds": POSITION_ITERATION, "pos_access": POSITION_ITERATION,
               "locate": LOCATE_CAPABLE, "size": INSERT_CAPABLE}[fn]
        self._require(cap, fn)
        dev = self._device()
        a = torch.as_tensor(a, dtype=torch.int64, device=dev).reshape(-1).contiguous()
        b = None if b is None else torch.as_tensor(b, dtype=torch.int64,
                                                   device=dev).reshape(-1).contiguous()
        o0 = torch.empty_like(a)
        o1 = torch.empty_like(a)
        d = self.descriptor()
        _lib.check(_lib.load().sl_level_query(ctypes.byref(d), _lib.FN_ID[fn], a.numel(),
                                              _lib.ptr(a), _lib.ptr(b), _lib.ptr(o0),
                                              _lib.ptr(o1), _lib.stream_handle()), fn)
        return o0, o1

    def _device(self):
        import torch

        for t in (self.crd, self.pos, self.offset):
            if t is not None:
                return t.device
        return torch.device("cuda")

    def _one(self, fn, a, b=None):
        o0, o1 = self.query(fn, [a], None if b is None else [b])
        return int(o0.item()), int(o1.item())

    # -- access functions (levels.py:215-282) --------------------------------

    def coord_bounds(self, prefix: Sequence[int]) -> Tuple[int, int]:
        return self._one("coord_bounds", prefix[-1] if len(prefix) else 0)

    def coord_access(self, parent_pos: int, coords: Sequence[int]) -> Tuple[int, bool]:
        p, f = self._one("coord_access", parent_pos, coords[-1])
        return p, bool(f)

    def pos_bounds(self, parent_pos: int) -> Tuple[int, int]:
        return self._one("pos_bounds", parent_pos)

    def pos_access(self, p: int, prefix: Sequence[int]) -> Tuple[int, bool]:
        c, f = self._one("pos_access", p, prefix[-1] if len(prefix) else 0)
        return c, bool(f)

    def locate(self, parent_pos: int, coords: Sequence[int]) -> Tuple[int, bool]:
        p, f = self._one("locate", parent_pos, coords[-1])
        return p, bool(f)

    def size(self, parent_size: int) -> int:
        return self._one("size", parent_size)[0]

    # -- assembly: insert (levels.py:286-338), bulk on the device -------------

    def insert_init(self, parent_size: int, size: int) -> None:
        import torch

        self._require(INSERT_CAPABLE, "insert_init")
        if self.kind is LevelKind.HASHED:
            self.crd = torch.empty(size, dtype=torch.int32, device=self._device())
            _lib.check(_lib.load().sl_hashed_insert_init(size, _lib.ptr(self.crd),
                                                         _lib.stream_handle()), "insert_init")

    def insert_coords(self, parent_pos, coords) -> None:
        """Bulk insert_coord for a hashed level: coordinate coords[q] into the
        segment of parent_pos[q].  Idempotent; raises HashSegmentFullError on
        overflow (levels.py:330-332)."""
        import torch

        self._require(INSERT_CAPABLE, "insert_coord")
        if self.kind is LevelKind.DENSE:
            return
        dev = self._device()
        coords = torch.as_tensor(coords, dtype=torch.int32, device=dev).reshape(-1).contiguous()
        pp = None if parent_pos is None else torch.as_tensor(
            parent_pos, dtype=torch.int32, device=dev).reshape(-1).contiguous()
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        # the exact table of sequential insert_coord calls in this order
        lib = _lib.load()
        nbytes = int(lib.sl_hashed_insert_ordered_workspace_bytes(coords.numel(), self.crd.numel()))
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _lib.check(lib.sl_hashed_insert_ordered(coords.numel(), _lib.ptr(pp), _lib.ptr(coords),
                                                self.w, self.crd.numel(), _lib.ptr(self.crd),
                                                _lib.ptr(err), _lib.ptr(ws), ws.numel(),
                                                _lib.stream_handle()), "insert_coord")
        if int(err.item()) != 0:
            raise HashSegmentFullError(
                f"hashed segment of width {self.w} is full")

    def insert_coord(self, p: int, coord: int) -> None:
        self._require(INSERT_CAPABLE, "insert_coord")
        if self.kind is LevelKind.HASHED:
            self.insert_coords([p // self.w], [coord])

    def insert_finalize(self, parent_size: int, size: int) -> None:
        self._require(INSERT_CAPABLE, "insert_finalize")

    # -- assembly: append (levels.py:342-394) ---------------------------------
    # Host-side staging of the sequential append protocol for API parity; the
    # hot path's append output (C = A + B) is produced in bulk by the
    # count/scan/fill kernels instead.

    def append_init(self, parent_size: int, size: int) -> None:
        self._require(APPEND_CAPABLE, "append_init")
        self._appended = []
        self._edges = [0] * (parent_size + 1) if self.kind is LevelKind.COMPRESSED else None
        self._last_edge_parent = -1

    def append_coord(self, p: int, coord: int) -> None:
        self._require(APPEND_CAPABLE, "append_coord")
        if self._appended is None:
            self._appended = []
        self._appended.append(int(coord))

    def append_edges(self, parent_pos: int, pbegin: int, pend: int) -> None:
        self._require(APPEND_CAPABLE, "append_edges")
        if self.kind is not LevelKind.COMPRESSED:
            return
        if self._edges is None:
            self._edges = [0]
        if parent_pos <= self._last_edge_parent:
            raise AssemblyError(f"append_edges parent position regressed: {parent_pos} after "
                                f"{self._last_edge_parent}")
        if parent_pos != self._last_edge_parent + 1:
            raise AssemblyError(f"append_edges skipped parent positions between "
                                f"{self._last_edge_parent} and {parent_pos}")
        if parent_pos + 1 < len(self._edges):
            self._edges[parent_pos + 1] = pend
        else:
            self._edges.append(pend)
        self._last_edge_parent = parent_pos

    def append_finalize(self, parent_size: int, size: int) -> None:
        self._require(APPEND_CAPABLE, "append_finalize")
        dev = self._device()
        if self._appended is not None:
            self.crd = _as_i32(self._appended, dev)
        if self.kind is LevelKind.COMPRESSED and self._edges is not None:
            self.pos = _as_i32(self._edges, dev)
        self._appended = self._edges = None
