"""GPU parity of the widened patterns: CSR x sparse-vector
(intersection) and SpMM (CSR x dense-2), against the reference's own
evaluate() outputs (tests/golden/widen.npz) and the oracle at larger sizes.
Bar: bit-exact (single ordered sums per output, no contraction)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1804_10112_b200 as sl  # noqa: E402
from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402
from conftest import load_cases  # noqa: E402


def cuda(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a).astype(dtype)), device="cuda")


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1).view(np.int64)


def test_widen_goldens_kernels_and_evaluate():
    seen = 0
    for name, c in load_cases("widen").items():
        n, m = int(c["nrows"]), int(c["ncols"])
        A = F.csr_storage(c["csr_pos"], c["csr_crd"], c["csr_vals"], (n, m))
        if name.startswith("spx"):
            y = K.spmv_csr_spx(n, m, cuda(c["csr_pos"], np.int32), cuda(c["csr_crd"], np.int32),
                               cuda(c["csr_vals"], np.float64), cuda(c["x_crd"], np.int32),
                               cuda(c["x_vals"], np.float64))
            assert np.array_equal(bits(y), bits(c["y"])), name
            x = F.sparse_vector_storage(c["x_crd"], c["x_vals"], m)
            y2 = sl.evaluate("y(i) = A(i,j) * x(j)", {"A": A, "x": x})
            assert np.array_equal(bits(y2.vals), bits(c["y"])), name
        else:
            Kc = int(c["K"])
            Y = K.spmm_csr(n, m, cuda(c["csr_pos"], np.int32), cuda(c["csr_crd"], np.int32),
                           cuda(c["csr_vals"], np.float64), cuda(c["X"], np.float64).view(m, Kc))
            assert np.array_equal(bits(Y), bits(c["Y"])), name
            X = F.dense_storage(np.asarray(c["X"]).reshape(m, Kc))
            for expr in ("Y(i,k) = A(i,j) * X(j,k)", "Y(i,k) = X(j,k) * A(i,j)"):
                Y2 = sl.evaluate(expr, {"A": A, "X": X})
                assert Y2.dims == (n, Kc)
                assert np.array_equal(bits(Y2.vals), bits(c["Y"])), (name, expr)
        seen += 1
    assert seen >= 16


@pytest.mark.parametrize("Kc", [1, 2, 5, 8, 16, 32, 40, 64])
def test_spmm_stencil_vs_oracle(orc, Kc):
    st = wl.stencil27(g=24, seed=4)
    n = st["nrows"]
    rng = np.random.default_rng(Kc)
    X = rng.uniform(-1, 1, (n, Kc))
    ref = orc.spmm_csr(n, Kc, st["pos"], st["crd"], st["vals"], X, threads=0)
    Y = K.spmm_csr(n, n, cuda(st["pos"], np.int32), cuda(st["crd"], np.int32),
                   cuda(st["vals"], np.float64), cuda(X, np.float64))
    assert np.array_equal(bits(Y), bits(ref))


def test_spmm_ragged_rows_vs_oracle(orc):
    """rows from 0 to 300 nonzeros (past every lane-group width)"""
    rng = np.random.default_rng(8)
    n, m, Kc = 700, 900, 12
    lens = rng.integers(0, 300, n)
    lens[::7] = 0
    pos = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=pos[1:])
    crd = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.uniform(-1, 1, len(crd))
    X = rng.uniform(-1, 1, (m, Kc))
    ref = orc.spmm_csr(n, Kc, pos.astype(np.int32), crd, vals, X, threads=0)
    Y = K.spmm_csr(n, m, cuda(pos, np.int32), cuda(crd, np.int32), cuda(vals, np.float64),
                   cuda(X, np.float64))
    assert np.array_equal(bits(Y), bits(ref))


@pytest.mark.parametrize("frac", [0.0, 0.01, 0.3, 1.0])
def test_spmv_spx_vs_oracle(orc, frac):
    d = wl.coo_spmv(n=50_000, nnz=500_000, seed=12)
    n, m = d["nrows"], d["ncols"]
    pos = wl.coo_to_csr_pos(d["rows"], n)
    rng = np.random.default_rng(int(frac * 100))
    keep = np.sort(rng.choice(m, int(m * frac), replace=False)).astype(np.int32)
    xv = rng.uniform(-1, 1, len(keep))
    ref, _ = orc.spmv_csr_spx(n, pos, d["cols"], d["vals"], keep, xv)
    y = K.spmv_csr_spx(n, m, cuda(pos, np.int32), cuda(d["cols"], np.int32),
                       cuda(d["vals"], np.float64), cuda(keep, np.int32), cuda(xv, np.float64))
    assert np.array_equal(bits(y), bits(ref))
