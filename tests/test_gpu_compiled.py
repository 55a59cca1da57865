"""GPU: `compile` / `compile_many` — `evaluate` bound once and replayed as a
CUDA graph with the streamed operands' host->device copies and the result's
device->host copy inside the graph.  Bars as for `evaluate`: SpMV bit-exact
against the oracle, MTTKRP within the condition-scaled 1e-12."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1804_10112_b200 as slb  # noqa: E402
from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
from paper_1804_10112_b200.errors import UnsupportedOutputError  # noqa: E402

EXPR = "y(i) = A(i,j) * x(j)"


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def _matrices(d):
    n, m = d["nrows"], d["ncols"]
    pos = wl.coo_to_csr_pos(d["rows"], n)
    e = wl.csr_to_ell(pos, d["cols"], d["vals"], n)
    return {"coo": F.coo_storage(d["rows"], d["cols"], d["vals"], (n, m)),
            "csr": F.csr_storage(pos, d["cols"], d["vals"], (n, m)),
            "ell": F.ell_storage(e["nslots"], e["crd"], e["vals"], (n, m))}


@pytest.mark.parametrize("fmt", ["coo", "csr", "ell"])
def test_compiled_spmv_streams_x_and_matches_oracle(orc, fmt):
    d = wl.coo_spmv(n=5000, nnz=60000, seed=11)
    n = d["nrows"]
    A = _matrices(d)[fmt]
    step = slb.compile(EXPR, {"A": A, "x": F.dense_storage(d["x"], device=None)})
    assert step.h2d_bytes == d["x"].nbytes and step.d2h_bytes == n * 8
    rng = np.random.default_rng(5)
    for trial in range(3):          # the graph re-reads the pinned host x every replay
        x = d["x"] if trial == 0 else rng.standard_normal(d["ncols"])
        step.operand("x").vals.copy_(torch.as_tensor(x))
        y = step.run().vals.numpy()
        ref, _ = orc.spmv_coo(n, d["rows"], d["cols"], d["vals"], x)
        assert np.array_equal(bits(y), bits(ref)), f"{fmt} trial {trial}"
        # and equals the eager call
        ye = slb.evaluate(EXPR, {"A": A, "x": F.dense_storage(x)}).vals
        assert np.array_equal(bits(y), bits(ye))


def test_compiled_pinned_operand_used_in_place():
    d = wl.coo_spmv(n=800, nnz=6000, seed=2)
    A = _matrices(d)["csr"]
    xh = torch.as_tensor(d["x"]).pin_memory()
    xs = F.dense_storage(xh, device=None)
    step = slb.compile(EXPR, {"A": A, "x": xs})
    assert step.operand("x").vals.data_ptr() == xs.vals.data_ptr()
    y0 = step.run().vals.clone()
    xh.mul_(2.0)                     # exact in binary: y doubles bit for bit
    y1 = step.run().vals
    assert np.array_equal(bits(y1), bits(2.0 * y0))


def test_compile_many_shares_streamed_operand_and_streams(orc):
    d = wl.coo_spmv(n=4000, nnz=50000, seed=4)
    n = d["nrows"]
    M = _matrices(d)
    x = F.dense_storage(d["x"], device=None)
    step = slb.compile_many([(EXPR, {"A": M["csr"], "x": x}, None),
                             (EXPR, {"A": M["ell"], "x": x}, None)])
    assert step.h2d_bytes == d["x"].nbytes            # one copy of the shared x
    assert step.d2h_bytes == 2 * n * 8
    ref, _ = orc.spmv_coo(n, d["rows"], d["cols"], d["vals"], d["x"])
    s = torch.cuda.Stream()
    for _ in range(2):
        y1, y2 = step(stream=s)
        step.synchronize()
        assert np.array_equal(bits(y1.vals), bits(ref))
        assert np.array_equal(bits(y2.vals), bits(ref))
        y1.vals.zero_(), y2.vals.zero_()


def test_compiled_device_result_and_dia(orc):
    d = wl.coo_spmv(n=3000, nnz=30000, seed=7)
    n, m = d["nrows"], d["ncols"]
    band = np.abs(d["cols"].astype(np.int64) - d["rows"]) <= 40
    dd = wl.dia_from_coo(d["rows"][band], d["cols"][band], d["vals"][band], n, m)
    ref, _ = orc.spmv_dia(n, m, dd["offsets"], dd["vals"], d["x"])
    step = slb.compile(EXPR, {"A": F.dia_storage(dd["offsets"], dd["vals"], (n, m)),
                              "x": F.dense_storage(d["x"], device=None)}, host_result=False)
    y = step.run()
    assert y.vals.is_cuda and step.d2h_bytes == 0
    assert np.array_equal(bits(y.vals), bits(ref))


def test_compiled_mttkrp_streams_factors(orc):
    t = wl.mttkrp(I=300, J=200, K=100, nnz=20000, R=32, seed=8)
    X = F.coo3_storage(t["i"], t["j"], t["k"], t["vals"], (300, 200, 100))
    Bh = F.dense_storage(t["B"], (200, 32), device=None)
    Ch = F.dense_storage(t["C"], (100, 32), device=None)
    step = slb.compile("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)", {"X": X, "B": Bh, "C": Ch})
    assert step.h2d_bytes == (200 + 100) * 32 * 8 and step.d2h_bytes == 300 * 32 * 8
    out = step.run().vals.numpy().reshape(300, 32)
    Ar, absA = orc.mttkrp_coo3(300, t["i"], t["j"], t["k"], t["vals"], t["B"], t["C"])
    ok, err = orc.within_condition(out, Ar, absA)
    assert ok, err
    eager = slb.evaluate("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)",
                         {"X": X, "B": F.dense_storage(t["B"], (200, 32)),
                          "C": F.dense_storage(t["C"], (100, 32))}).vals
    assert np.array_equal(bits(out.reshape(-1)), bits(eager))   # same kernels, same bits


def test_compile_rejects_data_dependent_outputs_and_host_sparse():
    ab = wl.add_ab(n=500, nnz_a=2000, nnz_b=2000, seed=3)
    A = F.csr_storage(ab["a_pos"], ab["a_crd"], ab["a_vals"], (500, 500))
    B = F.coo_storage(ab["b_rows"], ab["b_cols"], ab["b_vals"], (500, 500))
    with pytest.raises(UnsupportedOutputError):
        slb.compile("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B}, F.preset("csr"))
    d = wl.coo_spmv(n=500, nnz=4000, seed=2)
    x = F.dense_storage(d["x"])
    with pytest.raises(UnsupportedOutputError):
        slb.compile(EXPR, {"A": _matrices(d)["csr"], "x": x}, F.preset("hash-vector", width=1024))
    pos = wl.coo_to_csr_pos(d["rows"], 500)
    A_host = F.csr_storage(pos, d["cols"], d["vals"], (500, d["ncols"]), device=None)
    with pytest.raises(UnsupportedOutputError):
        slb.compile(EXPR, {"A": A_host, "x": x})
    # evaluate is unaffected afterwards
    y = slb.evaluate(EXPR, {"A": _matrices(d)["csr"], "x": x}).vals
    assert y.numel() == 500


def test_compiled_other_dense_output_patterns_match_evaluate():
    """SpMM with X streamed, TTV / TTM / MTTKRP over CSF with the dense operands
    streamed, CSR x hashed x (all operands resident): the replayed graph gives
    evaluate()'s bits, or compile refuses the statement outright."""
    st = wl.stencil27(g=12, seed=3)
    n = st["nrows"]
    A = F.csr_storage(st["pos"], st["crd"], st["vals"], (n, n))
    rng = np.random.default_rng(1)
    t = wl.mttkrp(I=60, J=50, K=40, nnz=6000, R=16, seed=5)
    csf = wl.coo3_to_csf(t["i"], t["j"], t["k"], None)
    X = F.csf_storage(csf["pos0"], csf["crd0"], csf["pos1"], csf["crd1"], csf["pos2"], csf["crd2"],
                      t["vals"], (60, 50, 40))
    d = wl.coo_spmv(n=3000, nnz=30000, seed=7)
    pos = wl.coo_to_csr_pos(d["rows"], 3000)
    Ah = F.csr_storage(pos, d["cols"], d["vals"], (3000, d["ncols"]))
    h = wl.hash_vector(n=d["ncols"], m=d["ncols"] // 2, width=4096, seed=9)
    cases = [
        ("Y(i,k) = A(i,j) * X(j,k)", {"A": A}, {"X": (rng.uniform(-1, 1, (n, 16)), (n, 16))}),
        ("Y(i,j) = X(i,j,k) * v(k)", {"X": X}, {"v": (rng.uniform(-1, 1, 40), (40,))}),
        ("Y(i,j,r) = X(i,j,k) * U(k,r)", {"X": X}, {"U": (rng.uniform(-1, 1, (40, 8)), (40, 8))}),
        ("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)", {"X": X},
         {"B": (t["B"], (50, 16)), "C": (t["C"], (40, 16))}),
        ("y(i) = A(i,j) * x(j)",
         {"A": Ah, "x": F.hash_vector_storage(h["crd"], h["vals"], d["ncols"], 4096)}, {}),
    ]
    for expr, resident, streamed in cases:
        host = {k: F.dense_storage(v, dims, device=None) for k, (v, dims) in streamed.items()}
        dev = {k: F.dense_storage(v, dims) for k, (v, dims) in streamed.items()}
        want = slb.evaluate(expr, {**resident, **dev}).vals
        try:
            step = slb.compile(expr, {**resident, **host})
        except UnsupportedOutputError:
            continue                      # refused: evaluate() is the path for it
        for _ in range(2):
            got = step.run().vals
            assert np.array_equal(bits(got), bits(want)), expr
