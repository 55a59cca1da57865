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
