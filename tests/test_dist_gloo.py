"""Multi-rank host logic on CPU (gloo, world size 2): nnz-balanced row/slice
partitioning, per-format shards, the x broadcast and the y all-gather.  Each
rank computes its block with the C oracle (test infrastructure) — on a GPU
box the same shards feed the sm_100a kernels."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

from paper_1804_10112_b200 import dist as D  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # SpMV (CSR): nnz-balanced row blocks, x broadcast from rank 0
        d = wl.coo_spmv(n=3000, nnz=40000, seed=5)
        pos = wl.coo_to_csr_pos(d["rows"], d["nrows"])
        bounds = D.balanced_row_blocks(pos, world)
        x = torch.as_tensor(d["x"]) if rank == 0 else torch.zeros(d["ncols"], dtype=torch.float64)
        D.replicate(x, src=0)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        lp, lc, lv = D.shard_csr(pos, d["cols"], d["vals"], r0, r1)
        y_loc = oracle.spmv_csr(r1 - r0, lp, lc, lv, x.numpy(), threads=1)
        y = D.gather_row_blocks(torch.as_tensor(y_loc), bounds)
        # MTTKRP (COO-3): slice blocks, factors replicated
        m = wl.mttkrp(I=300, J=200, K=100, nnz=30000, R=8, seed=6)
        sb = D.slice_blocks_coo3(m["i"], m["I"], world)
        s0, s1 = int(sb[rank]), int(sb[rank + 1])
        ii, jj, kk, vv = D.shard_coo3(m["i"], m["j"], m["k"], m["vals"], s0, s1)
        A_loc = oracle.mttkrp_coo3(s1 - s0, ii, jj, kk, vv, m["B"], m["C"], threads=1)
        A = D.gather_row_blocks(torch.as_tensor(A_loc.reshape(-1)), [b * m["R"] for b in sb])
        # A + B (CSR + COO -> CSR): row blocks, nnz totals all-gathered for the offsets
        ab = wl.add_ab(n=4000, nnz_a=16000, nnz_b=16000, seed=8)
        ab_bounds = D.balanced_row_blocks(ab["a_pos"], world)
        q0, q1 = int(ab_bounds[rank]), int(ab_bounds[rank + 1])
        (ap, ac, av), (br, bc, bv) = D.shard_add(ab["a_pos"], ab["a_crd"], ab["a_vals"],
                                                 ab["b_rows"], ab["b_cols"], ab["b_vals"], q0, q1)
        cp, cc, cv = oracle.add_csr(q1 - q0, ap, ac, av, bc, bv, b_rows=br)
        gp, gc, gv = D.concat_csr_blocks(torch.as_tensor(cp), torch.as_tensor(cc),
                                         torch.as_tensor(cv))
        t_max = D.max_over_ranks(float(rank + 1))
        t_sum = D.sum_over_ranks(float(rank + 1))
        if rank == 0:
            np.savez(out_dir / "dist.npz", y=y.numpy(), A=A.numpy(), bounds=bounds, sb=sb,
                     t_max=t_max, t_sum=t_sum, c_pos=gp.numpy(), c_crd=gc.numpy(),
                     c_vals=gv.numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_spmv_and_mttkrp(tmp_path, orc):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), tmp_path), nprocs=world, join=True)
    r = np.load(tmp_path / "dist.npz")
    d = wl.coo_spmv(n=3000, nnz=40000, seed=5)
    ref, _ = orc.spmv_coo(d["nrows"], d["rows"], d["cols"], d["vals"], d["x"])
    assert np.array_equal(r["y"].view(np.int64), ref.view(np.int64))
    m = wl.mttkrp(I=300, J=200, K=100, nnz=30000, R=8, seed=6)
    Aref, _ = orc.mttkrp_coo3(300, m["i"], m["j"], m["k"], m["vals"], m["B"], m["C"])
    # whole slices per rank: each output row is summed in the reference order
    assert np.array_equal(r["A"].view(np.int64), Aref.reshape(-1).view(np.int64))
    b = r["bounds"]
    assert b[0] == 0 and b[-1] == 3000 and (np.diff(b) > 0).all()
    assert float(r["t_max"]) == 2.0 and float(r["t_sum"]) == 3.0
    ab = wl.add_ab(n=4000, nnz_a=16000, nnz_b=16000, seed=8)
    rp, rc, rv = orc.add_csr(4000, ab["a_pos"], ab["a_crd"], ab["a_vals"], ab["b_cols"],
                             ab["b_vals"], b_rows=ab["b_rows"])
    assert np.array_equal(r["c_pos"], rp) and np.array_equal(r["c_crd"], rc)
    assert np.array_equal(r["c_vals"].view(np.int64), rv.view(np.int64))


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_shards_concatenate_to_the_whole(orc, parts):
    d = wl.coo_spmv(n=2000, nnz=30000, seed=7)
    n = d["nrows"]
    full, _ = orc.spmv_coo(n, d["rows"], d["cols"], d["vals"], d["x"])
    b = D.coo_row_blocks(d["rows"], n, parts)
    ys = []
    for p in range(parts):
        r0, r1 = int(b[p]), int(b[p + 1])
        rr, cc, vv = D.shard_coo(d["rows"], d["cols"], d["vals"], r0, r1)
        ys.append(orc.spmv_coo(r1 - r0, rr, cc, vv, d["x"], threads=1))
    assert np.array_equal(np.concatenate(ys).view(np.int64), full.view(np.int64))
    # nnz balance: no block exceeds its share by more than one row's worth
    pos = wl.coo_to_csr_pos(d["rows"], n)
    per = np.diff(pos[b])
    assert per.max() <= len(d["rows"]) / parts + np.diff(pos).max()
    # ELL and DIA shards
    e = wl.csr_to_ell(pos, d["cols"], d["vals"], n)
    ye = []
    for p in range(parts):
        r0, r1 = int(b[p]), int(b[p + 1])
        c, v = D.shard_ell(e["nslots"], e["crd"], e["vals"], n, r0, r1)
        ye.append(orc.spmv_ell(r1 - r0, e["nslots"], c, v, d["x"], threads=1))
    full_e, _ = orc.spmv_ell(n, e["nslots"], e["crd"], e["vals"], d["x"])
    assert np.array_equal(np.concatenate(ye).view(np.int64), full_e.view(np.int64))


def test_stencil_slabs_are_row_blocks():
    full = wl.stencil27(g=8, gz=16)
    parts = [wl.stencil27(g=8, gz=16, z0=z, z1=z + 4) for z in range(0, 16, 4)]
    assert np.array_equal(np.concatenate([p["crd"] for p in parts]), full["crd"])
    assert all(p["row0"] == 8 * 8 * z for p, z in zip(parts, range(0, 16, 4)))
    pos = np.concatenate([[0], np.cumsum([np.diff(p["pos"]).sum() for p in parts])])
    assert pos[-1] == full["pos"][-1]


# ---------------------------------------------------------------------------
# the public multi-GPU entry, evaluate_sharded, on two gloo ranks: device-side
# row blocks and shards, per-rank evaluation injected (the C oracle standing
# in for the sm_100a kernels), blocks all-gathered

def _oracle_eval(expr, inputs, out_format=None):
    """Per-rank evaluation by the C oracle for the patterns exercised below
    (test infrastructure; on a GPU box evaluate_sharded runs `evaluate`)."""
    import oracle

    from paper_1804_10112_b200 import engine as E
    from paper_1804_10112_b200 import formats as F

    p = E.plan_expression(expr, inputs, out_format)
    op = {role: inputs[name] for role, name in p.operands.items()}
    npy = lambda t: t.numpy()  # noqa: E731
    if p.pattern == "spmv":
        A, x = op["A"], npy(op["x"].vals)
        n, m = A.dims
        if p.kernel == "spmv_csr":
            y, _ = oracle.spmv_csr(n, npy(A.levels[1].pos), npy(A.levels[1].crd), npy(A.vals), x)
        elif p.kernel == "spmv_coo":
            y, _ = oracle.spmv_coo(n, npy(A.levels[0].crd), npy(A.levels[1].crd), npy(A.vals), x)
        elif p.kernel == "spmv_ell":
            y, _ = oracle.spmv_ell(n, A.levels[0].n, npy(A.levels[2].crd), npy(A.vals), x)
        else:
            y, _ = oracle.spmv_dia(n, m, npy(A.levels[1].offset), npy(A.vals), x)
        return F.dense_storage(torch.as_tensor(y), (n,), device="cpu")
    if p.pattern == "add":
        A, B = op["A"], op["B"]
        n = A.dims[0]
        cp, cc, cv = oracle.add_csr(n, npy(A.levels[1].pos), npy(A.levels[1].crd), npy(A.vals),
                                    npy(B.levels[1].crd), npy(B.vals), b_rows=npy(B.levels[0].crd))
        return F.csr_storage(cp, cc, cv, A.dims, device="cpu")
    if p.pattern == "mttkrp":
        X, Bm, Cm = op["X"], op["B"], op["C"]
        I, J, K = X.dims
        R = Bm.dims[1]
        Bv, Cv = npy(Bm.vals).reshape(J, R), npy(Cm.vals).reshape(K, R)
        if p.kernel == "mttkrp_csf":
            A, _ = oracle.mttkrp_csf(I, npy(X.levels[0].crd), npy(X.levels[1].pos),
                                     npy(X.levels[1].crd), npy(X.levels[2].pos),
                                     npy(X.levels[2].crd), npy(X.vals), Bv, Cv)
        else:
            A, _ = oracle.mttkrp_coo3(I, npy(X.levels[0].crd), npy(X.levels[1].crd),
                                      npy(X.levels[2].crd), npy(X.vals), Bv, Cv)
        return F.dense_storage(torch.as_tensor(A.reshape(-1)), (I, R), device="cpu")
    raise AssertionError(p.pattern)


def _sharded_worker(rank, world, port, out_dir):
    from paper_1804_10112_b200 import formats as F

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        d = wl.coo_spmv(n=3000, nnz=40000, seed=5)
        n, m = d["nrows"], d["ncols"]
        pos = wl.coo_to_csr_pos(d["rows"], n)
        x = F.dense_storage(torch.as_tensor(d["x"]), (m,), device="cpu")
        e = wl.csr_to_ell(pos, d["cols"], d["vals"], n)
        band = np.abs(d["cols"].astype(np.int64) - d["rows"]) <= 300
        dd = wl.dia_from_coo(d["rows"][band], d["cols"][band], d["vals"][band], n, m)
        mats = {"csr": F.csr_storage(pos, d["cols"], d["vals"], (n, m), device="cpu"),
                "coo": F.coo_storage(d["rows"], d["cols"], d["vals"], (n, m), device="cpu"),
                "ell": F.ell_storage(e["nslots"], e["crd"], e["vals"], (n, m), device="cpu"),
                "dia": F.dia_storage(dd["offsets"], dd["vals"], (n, m), device="cpu")}
        for name, A in mats.items():
            y = D.evaluate_sharded("y(i) = A(i,j) * x(j)", {"A": A, "x": x},
                                   local_eval=_oracle_eval)
            out[f"y_{name}"] = y.vals.numpy()
        # gather="p2p" needs the CUDA kernel's peer epilogue; with an injected
        # local evaluation it takes the collective gather, same result
        y = D.evaluate_sharded("y(i) = A(i,j) * x(j)", {"A": mats["csr"], "x": x},
                               gather="p2p", local_eval=_oracle_eval)
        out["y_p2p"] = y.vals.numpy()
        ab = wl.add_ab(n=4000, nnz_a=16000, nnz_b=16000, seed=8)
        A = F.csr_storage(ab["a_pos"], ab["a_crd"], ab["a_vals"], (4000, 4000), device="cpu")
        B = F.coo_storage(ab["b_rows"], ab["b_cols"], ab["b_vals"], (4000, 4000), device="cpu")
        C = D.evaluate_sharded("C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B}, F.preset("csr"),
                               local_eval=_oracle_eval)
        out["c_pos"], out["c_crd"] = C.levels[1].pos.numpy(), C.levels[1].crd.numpy()
        out["c_vals"] = C.vals.numpy()
        mt = wl.mttkrp(I=300, J=200, K=100, nnz=30000, R=8, seed=6)
        csf = wl.coo3_to_csf(mt["i"], mt["j"], mt["k"], None)
        Bf = F.dense_storage(torch.as_tensor(mt["B"].reshape(-1)), (200, 8), device="cpu")
        Cf = F.dense_storage(torch.as_tensor(mt["C"].reshape(-1)), (100, 8), device="cpu")
        Xs = {"coo3": F.coo3_storage(mt["i"], mt["j"], mt["k"], mt["vals"], (300, 200, 100),
                                     device="cpu"),
              "csf": F.csf_storage([0, len(csf["crd0"])], csf["crd0"], csf["pos1"], csf["crd1"],
                                   csf["pos2"], csf["crd2"], mt["vals"], (300, 200, 100),
                                   device="cpu")}
        for name, X in Xs.items():
            A_ = D.evaluate_sharded("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)",
                                    {"X": X, "B": Bf, "C": Cf}, local_eval=_oracle_eval)
            out[f"A_{name}"] = A_.vals.numpy()
        loc, (r0, r1) = D.evaluate_sharded("y(i) = A(i,j) * x(j)", {"A": mats["csr"], "x": x},
                                           gather=False, local_eval=_oracle_eval)
        out[f"block{rank}"] = np.array([r0, r1])
        allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, torch.tensor([r0, r1]))
        if rank == 0:
            out["blocks"] = torch.stack(allb).numpy()
            np.savez(out_dir / "sharded.npz", **out)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_evaluate_sharded(tmp_path, orc):
    world = 2
    mp.spawn(_sharded_worker, args=(world, _free_port(), tmp_path), nprocs=world, join=True)
    r = np.load(tmp_path / "sharded.npz")
    d = wl.coo_spmv(n=3000, nnz=40000, seed=5)
    n, m = d["nrows"], d["ncols"]
    ref, _ = orc.spmv_coo(n, d["rows"], d["cols"], d["vals"], d["x"])
    for name in ("csr", "coo", "ell", "p2p"):
        assert np.array_equal(r[f"y_{name}"].view(np.int64), ref.view(np.int64)), name
    band = np.abs(d["cols"].astype(np.int64) - d["rows"]) <= 300
    dd = wl.dia_from_coo(d["rows"][band], d["cols"][band], d["vals"][band], n, m)
    ref_d, _ = orc.spmv_dia(n, m, dd["offsets"], dd["vals"], d["x"])
    assert np.array_equal(r["y_dia"].view(np.int64), ref_d.view(np.int64))
    ab = wl.add_ab(n=4000, nnz_a=16000, nnz_b=16000, seed=8)
    rp, rc, rv = orc.add_csr(4000, ab["a_pos"], ab["a_crd"], ab["a_vals"], ab["b_cols"],
                             ab["b_vals"], b_rows=ab["b_rows"])
    assert np.array_equal(r["c_pos"], rp) and np.array_equal(r["c_crd"], rc)
    assert np.array_equal(r["c_vals"].view(np.int64), rv.view(np.int64))
    mt = wl.mttkrp(I=300, J=200, K=100, nnz=30000, R=8, seed=6)
    Aref, _ = orc.mttkrp_coo3(300, mt["i"], mt["j"], mt["k"], mt["vals"], mt["B"], mt["C"])
    for name in ("coo3", "csf"):        # whole slices per rank: the reference order per row
        assert np.array_equal(r[f"A_{name}"].view(np.int64), Aref.reshape(-1).view(np.int64)), name
    b = r["blocks"]
    assert b[0, 0] == 0 and b[0, 1] == b[1, 0] and b[1, 1] == n and 0 < b[0, 1] < n
