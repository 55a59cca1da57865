"""Format-property sweep: reference outputs for every preset x flag variant.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_sweep.py

For each supported expression pattern (SpMV, A + B, SpMM, MTTKRP, TTV, TTM,
INNERPROD) this varies one operand (or the output) over every preset of the
right order and, per preset, every configurable property flag of every level
flipped on its own (levels.py:46-92: full / ordered / unique), with the other
operands at their primary format and `fuse` both on and off.  Each variant's
tensor is built by the REFERENCE's own `assemble` (formats.py:361-501) from a
seeded coordinate list that repeats coordinates and arrives out of order (so a
non-unique or unordered level really holds duplicates / unsorted runs), and
the reference's `evaluate` (engine.py:739-764) gives either the output storage
and the `EvalStats.by_loop` visit counts, or the exception it raised.

The test (tests/test_gpu_sweep.py) rebuilds every case through this repo's API
and requires: the B200 path either raises UnsupportedMergeError /
UnsupportedOutputError (no kernel for that schedule) or produces exactly the
reference's output; where the reference raises, so must the repo.

Output: tests/golden/sweep.npz — one JSON manifest plus the flat arrays.
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import sparselevels as sl  # noqa: E402  (the reference)
from sparselevels import levels as rl  # noqa: E402
from sparselevels.engine import EvalStats  # noqa: E402

FLAGS = ("full", "ordered", "unique")

PRESETS = {
    1: ["dense", "sparse-vector", "hash-vector"],
    2: ["dense-2", "csr", "csc", "dcsr", "coo-soa", "coo-aos", "bcsr", "ell", "dia", "csb"],
    3: ["dense-3", "csf", "coo-3", "coo-3-aos", "mode-generic"],
}


def variants(name):
    """(tag, preset name, level flag overrides, reference format) per variant."""
    base = sl.preset(name)
    out = [("base", name, {}, base)]
    for k, spec in enumerate(base.levels):
        fixed = rl._FIXED[spec.kind]
        conf = [f for f in FLAGS if fixed[f] is None]
        for flag in conf:
            flags = {f: getattr(spec.props, f) for f in conf}
            flags[flag] = not flags[flag]
            new = rl.LevelSpec(spec.kind, rl.make_properties(spec.kind, **flags))
            fmt = dataclasses.replace(base, levels=base.levels[:k] + (new,) + base.levels[k + 1:])
            out.append((f"l{k}.{flag}={int(flags[flag])}", name, {str(k): flags}, fmt))
    return out


def primary(name):
    return ("base", name, {}, custom(name) if name.startswith("custom:") else sl.preset(name))


def custom(name):
    """custom:<kinds> formats beyond the presets, e.g. custom:hd = {hashed,
    dense} (a hashed first level over rows, dense columns)."""
    kinds = {"h": rl.hashed, "d": rl.dense, "c": rl.compressed}
    return sl.formats.simple_format([kinds[ch]() for ch in name.split(":", 1)[1]], name=name)


# ---------------------------------------------------------------------------
# seeded data: repeated coordinates, out-of-order entries, an explicit zero

def coords_for(dims, nnz, rng, dup_frac=0.25):
    n = len(dims)
    base = [tuple(int(rng.integers(0, d)) for d in dims) for _ in range(nnz)]
    ndup = max(1, int(nnz * dup_frac))
    for t in rng.choice(len(base), size=ndup, replace=True):
        base.append(base[int(t)])
    vals = rng.uniform(-1, 1, len(base)).round(6)
    vals[int(rng.integers(0, len(vals)))] = 0.0
    perm = rng.permutation(len(base))
    return [(base[int(p)], float(vals[int(p)])) for p in perm][: max(0, len(base))], n


def dense_entries(dims, rng):
    idx = np.indices(dims).reshape(len(dims), -1).T
    return [(tuple(int(c) for c in t), float(v))
            for t, v in zip(idx, rng.uniform(-1, 1, len(idx)).round(6))]


def make_tensor(fmt, dims, rng, dense=False, nnz=None):
    if dense or all(s.kind is rl.LevelKind.DENSE for s in fmt.levels):
        entries = dense_entries(dims, rng)
    else:
        nnz = nnz if nnz is not None else max(2, int(np.prod(dims) * 0.35))
        entries, _ = coords_for(dims, nnz, rng)
    return sl.assemble(fmt, tuple(dims), sl.CoordList(tuple(dims), entries))


def abs_dense(st):
    dims = st.dims
    out = np.zeros(int(np.prod(dims)) if dims else 1)
    for coords, v in sl.enumerate_storage(st).entries:
        out[int(np.ravel_multi_index(coords, dims)) if dims else 0] += abs(v)
    return out


# ---------------------------------------------------------------------------
# serialisation

class Pack:
    """All arrays concatenated into one int32 and one float64 pool; the
    manifest holds [offset, length] slices into them."""

    def __init__(self):
        self.pools = {np.int32: [], np.float64: []}
        self.size = {np.int32: 0, np.float64: 0}

    def arr(self, a, dtype):
        a = np.asarray(list(a), dtype=dtype)
        off = self.size[dtype]
        self.pools[dtype].append(a)
        self.size[dtype] += a.size
        return [int(off), int(a.size)]

    def arrays(self):
        return {"ints": np.concatenate(self.pools[np.int32] or [np.zeros(0, np.int32)]),
                "floats": np.concatenate(self.pools[np.float64] or [np.zeros(0)])}

    def storage(self, st, fmt_desc):
        lv = []
        for L in st.levels:
            lv.append({"n": int(L.n), "m": int(L.m), "w": int(L.w),
                       "pos": self.arr(L.pos, np.int32), "crd": self.arr(L.crd, np.int32),
                       "offset": self.arr(L.offset, np.int32), "crd_stride": int(L.crd_stride),
                       "crd_base": int(L.crd_base), "range_n": int(L.range_n)})
        return {"format": fmt_desc, "dims": [int(d) for d in st.dims], "levels": lv,
                "vals": self.arr(st.vals, np.float64)}


def fmt_desc(v):
    tag, name, flags, f = v
    d = {"preset": name, "tag": tag,
         "levels": {k: {f: bool(b) for f, b in fl.items()} for k, fl in flags.items()}}
    if f.hash_width:
        d["width"] = int(f.hash_width)
        d["tag"] = f"{tag},w={f.hash_width}"
    return d


def run_case(pack, cases, pattern, expr, ops, out, fuse, dims_of, rng):
    """ops: name -> variant; out: variant or None (default dense)."""
    inputs, desc = {}, {}
    try:
        for name, v in ops.items():
            dense = v[3].levels and any(s.props.full and s.kind is not rl.LevelKind.DENSE
                                        for s in v[3].levels)
            inputs[name] = make_tensor(v[3], dims_of[name], rng, dense=dense)
            desc[name] = fmt_desc(v)
    except sl.SparseLevelsError:
        return                                    # the variant cannot hold this data
    case = {"pattern": pattern, "expr": expr, "fuse": fuse,
            "inputs": {n: pack.storage(st, desc[n]) for n, st in inputs.items()},
            # |values| densified (duplicates' magnitudes summed): the bound
            # sum|terms| of the reassociated reductions is the same contraction
            "absdense": {n: pack.arr(abs_dense(st), np.float64) for n, st in inputs.items()},
            "out_format": None if out is None else fmt_desc(out)}
    stats = EvalStats()
    try:
        res = sl.evaluate(expr, inputs, None if out is None else out[3], fuse=fuse, stats=stats)
        case["result"] = pack.storage(res, case["out_format"])
        case["by_loop"] = [[k[0], k[1], int(v)] for k, v in stats.by_loop.items()]
    except sl.SparseLevelsError as e:
        case["error"] = type(e).__name__
    cases.append(case)


def sweep():
    pack, cases = Pack(), []
    rng = np.random.default_rng(20261020)
    fuses = (True, False)

    def all_variants(order):
        for name in PRESETS[order]:
            yield from variants(name)

    # ---- SpMV y(i) = A(i,j) * x(j)
    expr = "y(i) = A(i,j) * x(j)"
    dims = {"A": (6, 7), "x": (7,)}
    for fuse in fuses:
        for va in all_variants(2):
            run_case(pack, cases, "spmv", expr, {"A": va, "x": primary("dense")}, None, fuse,
                     dims, rng)
        for ab in ("csr", "coo-soa"):
            for vx in all_variants(1):
                run_case(pack, cases, "spmv", expr, {"A": primary(ab), "x": vx}, None, fuse,
                         dims, rng)
        for ab in ("csr", "coo-soa", "ell", "dia"):
            for vo in all_variants(1):
                run_case(pack, cases, "spmv", expr, {"A": primary(ab), "x": primary("dense")},
                         vo, fuse, dims, rng)

    # ---- C(i,j) = A(i,j) + B(i,j)
    expr = "C(i,j) = A(i,j) + B(i,j)"
    dims = {"A": (6, 7), "B": (6, 7)}
    csr = primary("csr")
    for fuse in fuses:
        for va in all_variants(2):
            run_case(pack, cases, "add", expr, {"A": va, "B": primary("coo-soa")}, csr, fuse,
                     dims, rng)
        for vb in all_variants(2):
            run_case(pack, cases, "add", expr, {"A": primary("csr"), "B": vb}, csr, fuse, dims,
                     rng)
        for vo in all_variants(2):
            run_case(pack, cases, "add", expr, {"A": primary("csr"), "B": primary("coo-soa")},
                     vo, fuse, dims, rng)

    # ---- SpMM Y(i,k) = A(i,j) * X(j,k)
    expr = "Y(i,k) = A(i,j) * X(j,k)"
    dims = {"A": (6, 7), "X": (7, 3)}
    for fuse in fuses:
        for va in all_variants(2):
            run_case(pack, cases, "spmm", expr, {"A": va, "X": primary("dense-2")}, None, fuse,
                     dims, rng)
        for vx in variants("dense-2"):
            run_case(pack, cases, "spmm", expr, {"A": primary("csr"), "X": vx}, None, fuse,
                     dims, rng)
        for vo in all_variants(2):
            run_case(pack, cases, "spmm", expr, {"A": primary("csr"), "X": primary("dense-2")},
                     vo, fuse, dims, rng)

    # ---- MTTKRP A(i,r) = X(i,j,k) * B(j,r) * C(k,r)
    expr = "A(i,r) = X(i,j,k) * B(j,r) * C(k,r)"
    dims = {"X": (4, 5, 6), "B": (5, 3), "C": (6, 3)}
    d2 = primary("dense-2")
    for fuse in fuses:
        for vx in all_variants(3):
            run_case(pack, cases, "mttkrp", expr, {"X": vx, "B": d2, "C": d2}, None, fuse, dims,
                     rng)
        for xb in ("coo-3", "csf"):
            for vb in variants("dense-2"):
                run_case(pack, cases, "mttkrp", expr, {"X": primary(xb), "B": vb, "C": d2}, None,
                         fuse, dims, rng)
                run_case(pack, cases, "mttkrp", expr, {"X": primary(xb), "B": d2, "C": vb}, None,
                         fuse, dims, rng)
            for vo in all_variants(2):
                run_case(pack, cases, "mttkrp", expr, {"X": primary(xb), "B": d2, "C": d2}, vo,
                         fuse, dims, rng)

    # ---- 3rd-order PLUS A(i,j,k) = X(i,j,k) + Z(i,j,k)
    expr = "A(i,j,k) = X(i,j,k) + Z(i,j,k)"
    dims = {"X": (4, 5, 6), "Z": (4, 5, 6)}
    c3 = primary("coo-3")
    for fuse in fuses:
        for vx in all_variants(3):
            run_case(pack, cases, "plus3", expr, {"X": vx, "Z": c3}, c3, fuse, dims, rng)
            run_case(pack, cases, "plus3", expr, {"X": c3, "Z": vx}, c3, fuse, dims, rng)
        for vo in all_variants(3):
            run_case(pack, cases, "plus3", expr, {"X": c3, "Z": c3}, vo, fuse, dims, rng)

    # ---- hashed outputs beyond SpMV: MTTKRP and SpMM into {hashed, dense},
    # A + B into {dense, hashed} (engine.py:292-317, levels.py:312-333)
    hd, dh = primary("custom:hd"), primary("custom:dh")
    for fuse in fuses:
        for xb in ("coo-3", "csf"):
            run_case(pack, cases, "mttkrp", "A(i,r) = X(i,j,k) * B(j,r) * C(k,r)",
                     {"X": primary(xb), "B": d2, "C": d2}, hd, fuse,
                     {"X": (4, 5, 6), "B": (5, 3), "C": (6, 3)}, rng)
        for ab in ("csr", "coo-soa"):
            run_case(pack, cases, "spmm", "Y(i,k) = A(i,j) * X(j,k)",
                     {"A": primary(ab), "X": d2}, hd, fuse, {"A": (6, 7), "X": (7, 3)}, rng)
            run_case(pack, cases, "add", "C(i,j) = A(i,j) + B(i,j)",
                     {"A": primary("csr"), "B": primary(ab)}, dh, fuse,
                     {"A": (6, 7), "B": (6, 7)}, rng)

    # ---- edge cases: empty operands and pinned hashed widths (too small ->
    # HashSegmentFullError in the reference, exactly full, roomy)
    def empty_case(pattern, expr, ops, out, dims_of):
        inputs = {n: sl.assemble(v[3], tuple(dims_of[n]), sl.CoordList(tuple(dims_of[n]), []))
                  for n, v in ops.items()}
        case = {"pattern": pattern, "expr": expr, "fuse": True,
                "inputs": {n: pack.storage(st, fmt_desc(ops[n])) for n, st in inputs.items()},
                "absdense": {n: pack.arr(abs_dense(st), np.float64) for n, st in inputs.items()},
                "out_format": None if out is None else fmt_desc(out)}
        stats = EvalStats()
        try:
            res = sl.evaluate(expr, inputs, None if out is None else out[3], stats=stats)
            case["result"] = pack.storage(res, case["out_format"])
            case["by_loop"] = [[k[0], k[1], int(v)] for k, v in stats.by_loop.items()]
        except sl.SparseLevelsError as e:
            case["error"] = type(e).__name__
        cases.append(case)

    d3 = {"X": (4, 5, 6), "Z": (4, 5, 6)}
    for o in ("coo-3", "csf", "dense-3"):
        empty_case("plus3", "A(i,j,k) = X(i,j,k) + Z(i,j,k)", {"X": c3, "Z": c3}, primary(o), d3)
    empty_case("ttv", "Y(i,j) = X(i,j,k) * v(k)", {"X": c3, "v": primary("dense")}, None,
               {"X": (4, 5, 6), "v": (6,)})
    empty_case("spmm", "Y(i,k) = A(i,j) * X(j,k)", {"A": primary("coo-soa"), "X": d2}, hd,
               {"A": (6, 7), "X": (7, 3)})
    for width in (2, 4, 8, 64):
        hdw = ("base", "custom:hd", {}, dataclasses.replace(custom("custom:hd"), hash_width=width))
        dhw = ("base", "custom:dh", {}, dataclasses.replace(custom("custom:dh"), hash_width=width))
        run_case(pack, cases, "mttkrp", "A(i,r) = X(i,j,k) * B(j,r) * C(k,r)",
                 {"X": primary("coo-3"), "B": d2, "C": d2}, hdw, True,
                 {"X": (4, 5, 6), "B": (5, 3), "C": (6, 3)}, rng)
        run_case(pack, cases, "add", "C(i,j) = A(i,j) + B(i,j)",
                 {"A": primary("csr"), "B": primary("coo-soa")}, dhw, True,
                 {"A": (6, 7), "B": (6, 7)}, rng)

    # ---- TTV Y(i,j) = X(i,j,k) * v(k), TTM Y(i,j,r) = X(i,j,k) * U(k,r)
    for fuse in fuses:
        e, dims = "Y(i,j) = X(i,j,k) * v(k)", {"X": (4, 5, 6), "v": (6,)}
        for vx in all_variants(3):
            run_case(pack, cases, "ttv", e, {"X": vx, "v": primary("dense")}, None, fuse, dims,
                     rng)
        for xb in ("coo-3", "csf"):
            for vv in all_variants(1):
                run_case(pack, cases, "ttv", e, {"X": primary(xb), "v": vv}, None, fuse, dims, rng)
            for vo in all_variants(2):
                run_case(pack, cases, "ttv", e, {"X": primary(xb), "v": primary("dense")}, vo,
                         fuse, dims, rng)
        e, dims = "Y(i,j,r) = X(i,j,k) * U(k,r)", {"X": (4, 5, 6), "U": (6, 3)}
        for vx in all_variants(3):
            run_case(pack, cases, "ttm", e, {"X": vx, "U": d2}, None, fuse, dims, rng)
        for xb in ("coo-3", "csf"):
            for vu in variants("dense-2"):
                run_case(pack, cases, "ttm", e, {"X": primary(xb), "U": vu}, None, fuse, dims, rng)
            for vo in all_variants(3):
                run_case(pack, cases, "ttm", e, {"X": primary(xb), "U": d2}, vo, fuse, dims, rng)
        # INNERPROD a() = X(i,j,k) * Z(i,j,k)
        e, dims = "a() = X(i,j,k) * Z(i,j,k)", {"X": (4, 5, 6), "Z": (4, 5, 6)}
        for vx in all_variants(3):
            run_case(pack, cases, "inner", e, {"X": vx, "Z": primary("coo-3")}, None, fuse, dims,
                     rng)
            run_case(pack, cases, "inner", e, {"X": primary("coo-3"), "Z": vx}, None, fuse, dims,
                     rng)
    return pack, cases


def main():
    pack, cases = sweep()
    manifest = json.dumps(cases, separators=(",", ":"))
    np.savez_compressed(HERE / "sweep.npz", manifest=np.array(manifest), **pack.arrays())
    ok = sum("result" in c for c in cases)
    print(f"sweep: {len(cases)} cases ({ok} evaluated, {len(cases) - ok} raised by the reference)")


if __name__ == "__main__":
    main()
