"""CPU-only tests of the host side: the C-ABI library loads and exports every
symbol include/sl_abi.h declares; the level property/capability model, the
format presets, the notation front end and the planner mirror the reference
(levels.py, formats.py, notation.py) — no kernel is launched here."""

import ctypes

import numpy as np
import pytest

from paper_1804_10112_b200 import _lib
from paper_1804_10112_b200 import engine as Eng
from paper_1804_10112_b200 import formats as F
from paper_1804_10112_b200 import levels as L
from paper_1804_10112_b200 import workloads as wl
from paper_1804_10112_b200.errors import (FormatError, NotationError, UnsupportedMergeError,
                                          UnsupportedOutputError, ValidationError)
from paper_1804_10112_b200.notation import Access, Add, Literal, Mul, parse, pretty, validate


# ---- C ABI --------------------------------------------------------------------

def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert set(syms) <= set(_lib.SIGNATURES)


def test_library_host_only_calls():
    lib = _lib.load()
    assert lib.sl_version() == 0x0100
    assert lib.sl_status_string(4) == b"hashed segment is full"
    assert lib.sl_status_string(999) == b"unknown status"
    # argument validation happens before any CUDA call
    assert lib.sl_spmv_coo_f64(-1, 0, 0, None, None, None, None, None, None, 0, None) == 1
    assert lib.sl_spmv_csr_f64(2**40, 1, 0, None, None, None, None, None, 0, None, 0, None) == 7
    assert lib.sl_hashed_locate(1, None, None, 0, None, None, None, 8, None) == 1
    assert lib.sl_mttkrp_coo3_f64(1, 1, 1, 200, 1, None, None, None, None, None, None, None, None,
                                  0, None) == 7
    # capability violations are rejected before launch (levels.py:197-199)
    d = _lib.SlLevel()
    d.kind = _lib.KIND_ID["range"]
    assert lib.sl_level_query(ctypes.byref(d), _lib.FN_ID["locate"], 1, None, None, None, None,
                              None) == 2
    assert lib.sl_mttkrp_workspace_bytes(40_000_000, 32) > 40_000_000 // 2048 * 2 * 32 * 8
    # widened entry points validate before launching too (1 = invalid, 7 = range, 8 = workspace)
    assert lib.sl_spmm_csr_f64(1, 1, -1, None, None, None, None, None, None) == 1
    assert lib.sl_spmm_csr_f64(2**40, 1, 4, None, None, None, None, None, None) == 7
    assert lib.sl_spmv_csr_spx_f64(1, 2**40, 0, None, None, None, 0, None, None, None, None, 0,
                                   None) == 7
    assert lib.sl_spmv_csr_spx_f64(1, 10, 0, ctypes.c_void_p(8), None, None, 0, None, None,
                                   ctypes.c_void_p(8), None, 0, None) == 8
    assert lib.sl_inner_coo3_f64(1, 1, 1, -1, None, None, None, None, 0, None, None, None, None,
                                 None, None, 0, None) == 1
    assert lib.sl_convert_coo_to_csr(1, 2**40, None, None, None) == 7
    assert lib.sl_hashed_slot_map(10, 0, None, None, 0, None) == 1
    assert lib.sl_spmv_csr_hashx_map_f64(1, 10, 0, None, None, None, 0, None, None, None, None,
                                         0, None) == 1
    assert lib.sl_csf_fiber_scatter_f64(-1, 1, 1, 0, 0, None, None, None, None, None, None) == 1
    assert lib.sl_add_csr_f64(-1, None, None, None, 0, None, None, None, None, None, None, None,
                              None, 0, None) == 1
    assert lib.sl_spmv_csr_workspace_bytes(10, 10, 0) == 0


def test_status_maps_to_reference_exceptions():
    from paper_1804_10112_b200 import errors as E
    for code, exc in ((2, E.UnsupportedCapabilityError), (4, E.HashSegmentFullError),
                      (5, E.UnsupportedMergeError), (6, E.UnsupportedOutputError)):
        with pytest.raises(exc):
            _lib.check(code)
    assert issubclass(E.HashSegmentFullError, E.AssemblyError)


# ---- level property model (test_levels.py:79-101) ------------------------------

def test_fixed_property_violations_rejected():
    for kind, flags in ((L.LevelKind.DENSE, dict(full=False)), (L.LevelKind.RANGE, dict(full=True)),
                        (L.LevelKind.HASHED, dict(ordered=True)),
                        (L.LevelKind.SINGLETON, dict(branchless=False)),
                        (L.LevelKind.OFFSET, dict(compact=True)),
                        (L.LevelKind.COMPRESSED, dict(branchless=True))):
        with pytest.raises(FormatError):
            L.make_properties(kind, **flags)
    with pytest.raises(FormatError):
        L.make_properties(L.LevelKind.DENSE, bogus=True)


def test_configurable_properties():
    p = L.make_properties(L.LevelKind.COMPRESSED, unique=False, full=True)
    assert not p.unique and p.full and p.compact and not p.branchless
    p = L.make_properties(L.LevelKind.DENSE)
    assert p.full and p.compact and p.ordered and p.unique
    assert L.make_properties(L.LevelKind.SINGLETON, branchless=True).branchless


def test_capability_sets_and_describe():
    assert L.dense().locate_capable and L.dense().insert_capable and L.dense().value_iterable
    assert L.hashed().locate_capable and L.hashed().position_iterable
    assert not L.range_level().locate_capable
    assert L.compressed().append_capable and L.singleton().append_capable
    assert not L.offset_level().append_capable
    assert L.compressed(unique=False).describe() == "compressed(~u)"
    assert L.LevelStorage(L.range_level(), n=3, device="cpu").kind is L.LevelKind.RANGE


def test_host_capability_errors_without_gpu():
    from paper_1804_10112_b200.errors import UnsupportedCapabilityError
    lv = L.LevelStorage(L.range_level(), n=4, m=6, offset=[0, -1], device="cpu")
    with pytest.raises(UnsupportedCapabilityError):
        lv.locate(0, [0, 0])
    with pytest.raises(UnsupportedCapabilityError):
        lv.pos_bounds(0)
    with pytest.raises(UnsupportedCapabilityError):
        L.LevelStorage(L.offset_level(), device="cpu").append_init(1, 0)


def test_host_append_protocol_errors():
    from paper_1804_10112_b200.errors import AssemblyError
    lv = L.LevelStorage(L.compressed(), device="cpu")
    lv.append_init(3, 0)
    lv.append_edges(0, 0, 0)
    lv.append_edges(1, 0, 0)
    with pytest.raises(AssemblyError):
        lv.append_edges(1, 0, 0)
    with pytest.raises(AssemblyError):
        lv.append_edges(3, 0, 0)


# ---- presets (formats.py:105-185) -------------------------------------------------

def test_presets_match_reference_table():
    expect = {
        "dense": "{dense}", "sparse-vector": "{compressed}", "hash-vector": "{hashed}",
        "csr": "{dense,compressed}", "csc": "{dense,compressed}@(1,0)",
        "dcsr": "{compressed,compressed}", "coo-soa": "{compressed(~u),singleton}",
        "coo-aos": "{compressed(~u),singleton}", "bcsr": "{dense,compressed,dense,dense}",
        "ell": "{dense,dense,singleton}", "dia": "{dense,range,offset}",
        "csb": "{dense,dense,compressed(~o,~u),singleton(~o)}",
        "csf": "{compressed,compressed,compressed}",
        "coo-3": "{compressed(~u),singleton(~u),singleton}",
        "mode-generic": "{compressed(~u),singleton,dense,dense}",
    }
    for name in F.PRESET_NAMES:
        assert F.preset(name).describe() == expect[name], name
    assert F.preset("coo").name == "coo-soa" and F.preset("hash", width=8).hash_width == 8
    with pytest.raises(FormatError):
        F.preset("nope")
    with pytest.raises(FormatError):
        F.preset("bcsr", block=0)


def test_format_classes():
    cls = {n: Eng.format_class(F.preset(n)) for n in F.PRESET_NAMES}
    assert cls["csr"] == "csr" and cls["coo-soa"] == "coo" and cls["ell"] == "ell"
    assert cls["dia"] == "dia" and cls["csf"] == "csf" and cls["coo-3"] == "coo3"
    assert cls["hash-vector"] == "hash1" and cls["dense"] == "dense1"
    assert cls["csc"].startswith("other") and cls["coo-aos"].startswith("other")
    assert cls["bcsr"].startswith("other")


# ---- notation (notation.py) ------------------------------------------------------

def test_parse_shapes_and_association():
    a = parse("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)")
    assert isinstance(a.rhs, Mul) and isinstance(a.rhs.left, Mul)
    assert a.rhs.left.left == Access("X", ("i", "j", "k"))
    a = parse("C(i,j) = A(i,j) - B(i,j)")
    assert isinstance(a.rhs, Add) and a.rhs.right.left == Literal(-1.0)
    assert pretty(parse("y(i)=A(i,j)*x(j)")) == "y(i) = A(i,j) * x(j)"
    assert pretty(parse("y(i) = 2 * (A(i,j) + B(i,j))")) == "y(i) = 2 * (A(i,j) + B(i,j))"
    for bad in ("y(i) = ", "y(i) = A(i,j) *", "y(i) A(i)", "y(i) = A(i,j) ) ", "y(1) = A(i)",
                "y(i) = A(i,j) $ x(j)"):
        with pytest.raises(NotationError):
            parse(bad)


def test_validate_rules():
    f2, f1 = F.preset("csr"), F.preset("dense")
    ok = validate(parse("y(i) = A(i,j) * x(j)"), {"A": (f2, (3, 4)), "x": (f1, (4,))})
    assert ok.reduction_vars == ("j",) and ok.var_extents == {"i": 3, "j": 4}
    for expr, b in (("y(i) = A(i,j) * x(j)", {"A": (f2, (3, 4)), "x": (f1, (5,))}),
                    ("y(i) = A(i,j) * z(j)", {"A": (f2, (3, 4))}),
                    ("y(i) = A(i,i)", {"A": (f2, (3, 3))}),
                    ("y(k) = A(i,j)", {"A": (f2, (3, 3))}),
                    ("y(i) = A(i)", {"A": (f2, (3, 3))}),
                    ("y(i) = A(i,j) + 2", {"A": (f2, (3, 3))})):
        with pytest.raises(ValidationError):
            validate(parse(expr), b)


# ---- planner: expression/format -> kernel ---------------------------------------------

def _st(fmt, dims):
    return F.TensorStorage(F.preset(fmt), dims, [], np.zeros(1))


def test_plan_dispatch_and_errors():
    def plan(expr, ins, out=None):
        a = parse(expr)
        b = {n: (s.format, s.dims) for n, s in ins.items()}
        c = validate(a, b)
        of = out or F.preset("dense", order=len(a.lhs.ivars))
        return Eng.plan(c, b, of, tuple(c.var_extents[v] for v in a.lhs.ivars))

    x = _st("dense", (4,))
    for fmt in ("coo-soa", "csr", "ell", "dia"):
        p = plan("y(i) = A(i,j) * x(j)", {"A": _st(fmt, (3, 4)), "x": x})
        assert p.kernel == "spmv_" + Eng.format_class(F.preset(fmt))
    assert plan("y(i) = x(j) * A(i,j)", {"A": _st("csr", (3, 4)), "x": x}).kernel == "spmv_csr"
    assert plan("y(i) = A(i,j) * x(j)", {"A": _st("csr", (3, 4)),
                                         "x": _st("hash-vector", (4,))}).kernel == "spmv_csr_hashx"
    with pytest.raises(UnsupportedMergeError):
        plan("y(i) = A(i,j) * x(j)", {"A": _st("csc", (3, 4)), "x": x})
    with pytest.raises(UnsupportedMergeError):
        plan("y(j) = A(i,j) * x(i)", {"A": _st("csr", (4, 4)), "x": x})
    with pytest.raises(UnsupportedOutputError):
        plan("y(i) = A(i,j) * x(j)", {"A": _st("csr", (3, 4)), "x": x}, F.preset("sv"))
    A, B = _st("csr", (3, 4)), _st("coo-soa", (3, 4))
    p = plan("C(i,j) = B(i,j) + A(i,j)", {"A": A, "B": B}, F.preset("csr"))
    assert p.kernel == "add_csr_coo_csr" and p.operands == {"A": "A", "B": "B"}
    assert plan("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": _st("csr", (3, 4))},
                F.preset("csr")).kernel == "add_csr_csr_csr"
    assert plan("C(i,j) = A(i,j) + B(i,j)", {"A": B, "B": B},
                F.preset("coo-soa")).kernel == "add_coo_coo_coo"
    with pytest.raises(UnsupportedOutputError):
        plan("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B})
    with pytest.raises(UnsupportedMergeError):
        plan("C(i,j) = A(i,j) + B(i,j)", {"A": _st("ell", (3, 4)), "B": B}, F.preset("csr"))
    X, Bd, Cd = _st("coo-3", (5, 6, 7)), _st("dense-2", (6, 3)), _st("dense-2", (7, 3))
    for expr in ("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)", "A(i,r) = B(j,r) * X(i,j,k) * C(k,r)",
                 "A(i,r) = C(k,r) * (X(i,j,k) * B(j,r))"):
        assert plan(expr, {"X": X, "B": Bd, "C": Cd}).kernel == "mttkrp_coo3"
    assert plan("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)",
                {"X": _st("csf", (5, 6, 7)), "B": Bd, "C": Cd}).kernel == "mttkrp_csf"
    with pytest.raises(UnsupportedMergeError):   # different association: (B*C)*X
        plan("A(i,r) = X(i,j,k) * (B(j,r) * C(k,r))", {"X": X, "B": Bd, "C": Cd})


# ---- generators --------------------------------------------------------------------------

def test_generators_hit_exact_sizes():
    d = wl.coo_spmv(n=2000, nnz=20000, seed=1)
    assert len(d["rows"]) == 20000
    keys = d["rows"].astype(np.int64) * d["ncols"] + d["cols"]
    assert (np.diff(keys) > 0).all()
    s = wl.stencil27(g=8)
    assert len(s["crd"]) == (3 * 8 - 2) ** 3 and s["pos"][-1] == len(s["crd"])
    slab = wl.stencil27(g=8, gz=16, z0=8, z1=16)
    assert slab["nrows"] == 8 * 8 * 8 and slab["ncols"] == 8 * 8 * 16 and slab["row0"] == 512
    a = wl.add_ab(n=3000, nnz_a=15000, nnz_b=15000, seed=2)
    assert len(a["a_crd"]) == 15000 and len(a["b_cols"]) == 15000
    assert 0 < a["overlap"] < 15000 * 0.2
    m = wl.mttkrp(I=100, J=80, K=60, nnz=5000, R=4, seed=3)
    key = (m["i"].astype(np.int64) * 80 + m["j"]) * 60 + m["k"]
    assert len(key) == 5000 and (np.diff(key) > 0).all() and (m["vals"] > 0).all()


def test_plan_cache_identity_fast_path(monkeypatch):
    """evaluate()'s identity plan cache: a repeated call with the same format
    objects reuses the plan; other dims, other formats (equal or not) and an
    explicit out_format plan correctly (no GPU: _run is stubbed to return the
    plan)."""
    monkeypatch.setattr(Eng, "_run", lambda p, inputs, stats: p)
    Eng._FAST_CACHE.clear()
    pos, crd, vals = np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.ones(2)
    A = F.csr_storage(pos, crd, vals, (2, 2), device=None)
    x = F.dense_storage(np.ones(2), device=None)
    expr = "y(i) = A(i,j) * x(j)"
    p1 = Eng.evaluate(expr, {"A": A, "x": x})
    assert p1.kernel == "spmv_csr" and len(Eng._FAST_CACHE) == 1
    assert Eng.evaluate(expr, {"A": A, "x": x}) is p1             # identity hit
    A3 = F.csr_storage(np.array([0, 1, 2, 2], np.int32), crd, vals, (3, 2), device=None)
    p3 = Eng.evaluate(expr, {"A": A3, "x": x})
    assert p3 is not p1 and p3.out_dims == (3,)                 # dims are part of the key
    C = F.coo_storage(np.array([0, 1], np.int32), crd, vals, (2, 2), device=None)
    assert Eng.evaluate(expr, {"A": C, "x": x}).kernel == "spmv_coo"
    hv = F.preset("hash-vector")
    ph = Eng.evaluate(expr, {"A": A, "x": x}, out_format=hv)
    assert ph.out_format is hv and ph is not p1
    assert Eng.evaluate(expr, {"A": A, "x": x}) is p1


# ---- compile: no CPU fallback ---------------------------------------------------

def test_compile_without_a_gpu_raises_device_error():
    import torch

    import paper_1804_10112_b200 as slb
    from paper_1804_10112_b200.errors import DeviceError

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    x = F.dense_storage(np.ones(4), device=None)
    with pytest.raises(DeviceError):
        slb.compile("y(i) = x(i)", {"x": x})
    with pytest.raises(ValueError):
        slb.compile_many([])
