"""CPU: the planner against the reference over the format-property sweep
(tests/golden/sweep.npz): every case the reference rejects is rejected here
too, and for every case the B200 path accepts, the loop-visit counts it
reports (EvalStats.by_loop) equal the reference's — computed here with the
inputs on the host (the GPU test repeats it through `evaluate`)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import sweep_util as su  # noqa: E402

import paper_1804_10112_b200 as slb  # noqa: E402
from paper_1804_10112_b200 import engine as E  # noqa: E402

CASES = list(enumerate(su.cases()))


def _plan(case, inputs):
    return slb.plan_expression(case["expr"], inputs, su.fmt(case["out_format"]),
                               fuse=case["fuse"])


# raised by the reference while executing (a full hashed segment): the
# planner cannot know; the GPU sweep checks that `evaluate` raises them too
RUNTIME_ERRORS = {"HashSegmentFullError"}


def test_rejected_by_reference_rejected_here():
    for i, case in CASES:
        if "error" not in case or case["error"] in RUNTIME_ERRORS:
            continue
        with pytest.raises(slb.SparseLevelsError):
            _plan(case, su.inputs(case, "cpu"))


def test_loop_counts_match_reference():
    checked = 0
    for i, case in CASES:
        if "error" in case:
            continue
        inputs = su.inputs(case, "cpu")
        try:
            p = _plan(case, inputs)
        except (slb.UnsupportedMergeError, slb.UnsupportedOutputError):
            continue
        ops = {role: inputs[name] for role, name in p.operands.items()}
        if any(not s.format.levels[-1].props.unique and E.format_class(s.format) == "csr"
               for s in ops.values()):
            continue                        # grouping a non-unique CSR runs a kernel
        got = {k: v for k, v in E._loop_counts(p, ops, None).items() if v}
        assert got == {(v, lab): n for v, lab, n in case["by_loop"]}, su.case_id(i, case)
        checked += 1
    assert checked >= 300


def _csr_group(orc, nrows, pos, crd, vals):
    """Grouped (engine.py:107-149) CSR: the identity copy, A+B with A empty."""
    z = np.zeros(nrows + 1, np.int32)
    return orc.add_csr(nrows, z, z[:0], np.zeros(0), crd, vals, b_pos=pos)


def _host(st):
    lv = st.levels
    return [None if t is None else t.numpy() for t in
            [getattr(l, a) for l in lv for a in ("pos", "crd")]], st.vals.numpy()


def _bits(a):
    a = np.ascontiguousarray(a, np.float64)
    b = a.view(np.int64).copy()
    b[a == 0.0] = 0
    return b


def test_oracle_matches_reference_on_sweep(orc):
    """The C oracle (the GPU tests' checker) restates the grouped semantics:
    for every SpMV / A + B / INNERPROD variant the B200 path accepts, the
    oracle's output equals the reference's, bit for bit."""
    checked = 0
    for i, case in CASES:
        if "error" in case or case["pattern"] not in ("spmv", "add", "inner"):
            continue
        inputs = su.inputs(case, "cpu")
        try:
            p = _plan(case, inputs)
        except (slb.UnsupportedMergeError, slb.UnsupportedOutputError):
            continue
        ops = {role: inputs[name] for role, name in p.operands.items()}
        ref = case["result"]
        if p.pattern == "spmv" and E.format_class(p.out_format) == "dense1":
            A, x = ops["A"], ops["x"].vals.numpy()
            n, m = A.dims
            av = A.vals.numpy()
            if p.kernel == "spmv_coo":
                r, c = A.levels[0].crd.numpy(), A.levels[1].crd.numpy()
                y, _ = orc.spmv_coo(n, r, c, av[:len(c)], x)
            elif p.kernel in ("spmv_csr", "spmv_coo_grouped"):
                if p.kernel == "spmv_csr":
                    pos, crd = A.levels[1].pos.numpy(), A.levels[1].crd.numpy()
                else:
                    crd = A.levels[1].crd.numpy()
                    pos = np.searchsorted(A.levels[0].crd.numpy(), np.arange(n + 1)).astype(
                        np.int32)
                pos, crd, av = _csr_group(orc, n, pos, crd, av[:len(crd)])
                y, _ = orc.spmv_csr(n, pos, crd, av, x)
            elif p.kernel == "spmv_ell":
                S = A.levels[0].n
                y, _ = orc.spmv_ell(n, S, A.levels[2].crd.numpy(), av[:S * n], x)
            elif p.kernel == "spmv_dia":
                offs = A.levels[1].offset.numpy()
                y, _ = orc.spmv_dia(n, m, offs, av[:len(offs) * n], x)
            else:
                continue
            want = su.floats(ref["vals"])[:n]
            assert np.array_equal(_bits(y), _bits(want)), su.case_id(i, case)
        elif p.pattern == "add" and p.kernel.endswith("_csr"):
            A, B = ops["A"], ops["B"]
            n = A.dims[0]

            def as_csr(st):
                v = st.vals.numpy()
                if E.format_class(st.format) == "csr":
                    pos, crd = st.levels[1].pos.numpy(), st.levels[1].crd.numpy()
                else:
                    crd = st.levels[1].crd.numpy()
                    pos = np.searchsorted(st.levels[0].crd.numpy(), np.arange(n + 1)).astype(
                        np.int32)
                return pos, crd, v[:len(crd)]

            apos, acrd, av = _csr_group(orc, n, *as_csr(A))
            bpos, bcrd, bv = as_csr(B)
            cpos, ccrd, cv = orc.add_csr(n, apos, acrd, av, bcrd, bv, b_pos=bpos)
            assert np.array_equal(cpos, su.ints(ref["levels"][1]["pos"])), su.case_id(i, case)
            assert np.array_equal(ccrd, su.ints(ref["levels"][1]["crd"])), su.case_id(i, case)
            want = su.floats(ref["vals"])[:len(cv)]
            assert np.array_equal(_bits(cv), _bits(want)), su.case_id(i, case)
        elif p.pattern == "inner":
            X, Z = ops["X"], ops["Z"]
            d = lambda st: {"i": st.levels[0].crd.numpy(), "j": st.levels[1].crd.numpy(),
                            "k": st.levels[2].crd.numpy(),
                            "vals": st.vals.numpy()[:st.levels[2].crd.numel()]}
            a, _ = orc.inner_coo3(d(X), d(Z))
            want = su.floats(ref["vals"])[:1]
            assert np.array_equal(_bits(np.array([a])), _bits(want)), su.case_id(i, case)
        else:
            continue
        checked += 1
    assert checked >= 140
