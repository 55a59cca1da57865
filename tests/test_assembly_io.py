"""Host-side data formats around the hot path: assembly of
coordinate lists into every in-scope format and the Matrix Market / FROSTT
readers, against the reference's own assemble() / read_mtx() / read_tns()
outputs (tests/golden/assembly.npz, io.npz).  CPU only."""

import numpy as np
import pytest

from conftest import load_cases
from paper_1804_10112_b200 import assembly as A
from paper_1804_10112_b200 import io as IO
from paper_1804_10112_b200.errors import AssemblyError

FMTS = {"coo_soa": "coo-soa", "csr": "csr", "ell": "ell", "dia": "dia", "coo_3": "coo-3",
        "csf": "csf", "sparse_vector": "sparse-vector", "hash_vector": "hash-vector",
        "dense": "dense"}


def _np(t):
    return t.numpy() if hasattr(t, "numpy") else np.asarray(t)


def _bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.int64)


def test_assembly_matches_reference():
    from paper_1804_10112_b200.formats import preset
    checked = 0
    for name, c in load_cases("assembly").items():
        dims = tuple(int(d) for d in c["dims"])
        data = A.CoordList(dims, c["coords"], c["vals"])
        prefixes = sorted({k.split("_l")[0].rsplit("_vals", 1)[0] for k in c
                           if k.endswith("_vals") and k != "vals"})
        for pre in prefixes:
            fmt = preset(FMTS[pre], slots=12) if name == "asm_ell_declared" else \
                preset(FMTS[pre], len(dims)) if FMTS[pre] == "dense" else preset(FMTS[pre])
            st = A.assemble(fmt, dims, data, device=None)
            want_vals = c[f"{pre}_vals"]
            got_vals = _np(st.vals)
            # the reference pads vals to at least one slot; compare the stored prefix
            assert np.array_equal(_bits(got_vals), _bits(want_vals[:len(got_vals)])), (name, pre)
            assert (want_vals[len(got_vals):] == 0).all(), (name, pre)
            for key in c:
                if not key.startswith(pre + "_l"):
                    continue
                k, attr = key[len(pre) + 2:].split("_", 1)
                lv = st.levels[int(k)]
                got = getattr(lv, attr)
                got = int(got) if attr in ("n", "w") else _np(got)
                if attr in ("n", "w"):
                    assert got == int(c[key]), (name, key)
                else:
                    assert np.array_equal(np.asarray(got).astype(np.int64),
                                          np.asarray(c[key]).astype(np.int64)), (name, key)
            checked += 1
    assert checked >= 10


def test_assembly_errors():
    from paper_1804_10112_b200.formats import preset
    with pytest.raises(AssemblyError):
        A.assemble("csr", (2, 2), A.CoordList((2, 2), [[2, 0]], [1.0]), device=None)
    with pytest.raises(AssemblyError):
        A.assemble(preset("ell", slots=1), (2, 3), A.CoordList((2, 3), [[0, 0], [0, 1]], [1., 2.]),
                   device=None)
    with pytest.raises(AssemblyError):
        A.assemble("dia", (3, 3), A.CoordList((3, 3), [[0, 2]], [1.0]), diagonals=[0, 1],
                   device=None)


def test_canonicalize_sums_in_input_order():
    # 1e16 + 1 - 1e16 in input order is 0 -> dropped; a signed zero is dropped too
    d = A.CoordList((3,), [[1], [1], [1], [2]], [1e16, 1.0, -1e16, -0.0])
    c = A.canonicalize(d)
    assert c.nnz == 0


@pytest.mark.parametrize("name", ["mtx_real", "mtx_pattern", "mtx_int", "mtx_bad_sym",
                                  "mtx_bad_count", "mtx_out_of_range", "mtx_no_header",
                                  "mtx_bad_field", "tns_basic", "tns_bad_order", "tns_zero_based"])
def test_readers_match_reference(tmp_path, name):
    c = load_cases("io")[name]
    kind = str(c["kind"])
    path = tmp_path / f"{name}.{kind}"
    path.write_text(str(c["text"]))
    reader = IO.read_mtx if kind == "mtx" else IO.read_tns
    if "error" in c:
        with pytest.raises(IO.FileFormatError) as ei:
            reader(str(path))
        assert str(ei.value).replace(str(tmp_path) + "/", "") == str(c["error"])
        return
    cl = reader(str(path))
    assert cl.dims == tuple(int(d) for d in c["dims"])
    assert np.array_equal(cl.coords, c["coords"])
    assert np.array_equal(_bits(cl.vals), _bits(c["vals"]))


def test_writers_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    d2 = A.CoordList((7, 5), np.stack([rng.integers(0, 7, 20), rng.integers(0, 5, 20)], 1),
                     rng.uniform(-1, 1, 20))
    IO.write_mtx(d2, str(tmp_path / "a.mtx"))
    r2 = IO.read_mtx(str(tmp_path / "a.mtx"))
    assert r2.dims == d2.dims and np.array_equal(r2.coords, d2.coords)
    assert np.array_equal(_bits(r2.vals), _bits(d2.vals))
    d3 = A.CoordList((4, 3, 6), np.stack([rng.integers(0, 4, 15), rng.integers(0, 3, 15),
                                          rng.integers(0, 6, 15)], 1), rng.uniform(-1, 1, 15))
    IO.write_tns(d3, str(tmp_path / "a.tns"))
    r3 = IO.read_tns(str(tmp_path / "a.tns"), dims=d3.dims)
    assert r3.dims == d3.dims and np.array_equal(r3.coords, d3.coords)
    assert np.array_equal(_bits(r3.vals), _bits(d3.vals))
