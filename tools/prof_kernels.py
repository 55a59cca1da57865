#!/usr/bin/env python
"""Run each hot-path kernel at its BASELINE size a few times (L2 flushed
before each launch) — the target for `ncu` captures and a quick CUDA-event
table with and without the flush.

    python tools/prof_kernels.py [--reps N] [--only coo,csr,...] [--no-table]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--no-table", action="store_true")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    jobs = {}

    def want(k):
        return not only or k in only

    def d1():
        d = wl.coo_spmv()
        n, m = d["nrows"], d["ncols"]
        r, c, v, x = T(d["rows"]), T(d["cols"]), T(d["vals"]), T(d["x"])
        y = torch.empty(n, dtype=torch.float64, device=dev)
        pos = T(wl.coo_to_csr_pos(d["rows"], n))
        jobs["coo"] = (35_200_000, lambda: K.spmv_coo(n, m, r, c, v, x, y))
        jobs["csr_d1"] = (4 * (n + 1) + 12 * len(d["rows"]) + 16 * n,
                          lambda: K.spmv_csr(n, m, pos, c, v, x, y))
        for tag, w in (("hashx", 131_072), ("hashx_wdef", 524_288)):
            h = wl.hash_vector(width=w)
            hc, hv = T(h["crd"]), T(h["vals"])
            jobs[tag] = (4 * (n + 1) + 12 * len(d["rows"]) + 8 * n + 12 * w,
                         lambda hc=hc, hv=hv, w=w: K.spmv_csr_hashx(n, pos, c, v, w, hc, hv, y))
            hws = torch.empty(int(K.L().sl_spmv_csr_hashx_map_workspace_bytes(m, w)),
                              dtype=torch.uint8, device=dev)
            jobs[tag + "_map"] = (4 * (n + 1) + 12 * len(d["rows"]) + 8 * n + 12 * w,
                                  lambda hc=hc, hv=hv, w=w, hws=hws: K.spmv_csr_hashx(
                                      n, pos, c, v, w, hc, hv, y, n=m, ws=hws))

    def d2():
        s = wl.stencil27()
        n = s["nrows"]
        e = wl.csr_to_ell(s["pos"], s["crd"], s["vals"], n)
        p, c, v, x = T(s["pos"]), T(s["crd"]), T(s["vals"]), T(s["x"])
        ec, ev = T(e["crd"]), T(e["vals"])
        y = torch.empty(n, dtype=torch.float64, device=dev)
        bc = 4 * (n + 1) + 12 * len(s["crd"]) + 16 * n
        jobs["csr"] = (bc, lambda: K.spmv_csr(n, n, p, c, v, x, y, variant=0))
        rr = T(np.repeat(np.arange(n, dtype=np.int32), np.diff(s["pos"])))
        jobs["coo_st"] = (16 * len(s["crd"]) + 16 * n,
                          lambda: K.spmv_coo(n, n, rr, c, v, x, y))
        jobs["csr_merge"] = (bc, lambda: K.spmv_csr(n, n, p, c, v, x, y, variant=2))
        if K.L().sl_build_features() & 1:     # A/B build (SL_BUILD_ALT=1) only
            jobs["csr_vec"] = (bc, lambda: K.spmv_csr(n, n, p, c, v, x, y, variant=1))
            jobs["csr_warp"] = (bc, lambda: K.spmv_csr(n, n, p, c, v, x, y, variant=3))
        for Kc in (4, 16, 32):
            Xd = torch.rand((n, Kc), dtype=torch.float64, device=dev)
            Yd = torch.empty((n, Kc), dtype=torch.float64, device=dev)
            jobs[f"spmm{Kc}"] = (4 * (n + 1) + 12 * len(s["crd"]) + 16 * n * Kc,
                                 lambda Xd=Xd, Yd=Yd: K.spmm_csr(n, n, p, c, v, Xd, Yd))
        jobs["ell"] = (12 * 27 * n + 16 * n, lambda: K.spmv_ell(n, n, 27, ec, ev, x, y))

    def d3():
        g = wl.dia7()
        n = g["nrows"]
        gv, gx = T(g["vals"]), T(g["x"])
        yd = torch.empty(n, dtype=torch.float64, device=dev)
        jobs["dia"] = (150_730_764, lambda: K.spmv_dia(n, n, g["offsets"], gv, gx, yd))

    def d4():
        a = wl.add_ab()
        n = a["nrows"]
        ap_, ac, av = T(a["a_pos"]), T(a["a_crd"]), T(a["a_vals"])
        br, bc_, bv = T(a["b_rows"]), T(a["b_cols"]), T(a["b_vals"])
        jobs["add"] = (262_406_292, lambda: K.add_csr(n, ap_, ac, av, bc_, bv, b_rows=br,
                                                      sync=False))

    def d5():
        mt = wl.mttkrp()
        csf = wl.coo3_to_csf(mt["i"], mt["j"], mt["k"], None)
        I, J, Kd, R = mt["I"], mt["J"], mt["K"], mt["R"]
        nnz = len(mt["i"])
        ti, tj, tk, tv = T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"])
        Bt, Ct = T(mt["B"]), T(mt["C"])
        c0, p1, c1, p2, c2 = (T(csf[k]) for k in ("crd0", "pos1", "crd1", "pos2", "crd2"))
        A = torch.empty((I, R), dtype=torch.float64, device=dev)
        ws = torch.empty(int(K.L().sl_mttkrp_workspace_bytes(nnz, R)), dtype=torch.uint8,
                         device=dev)
        jobs["mttkrp_coo"] = (811_520_000, lambda: K.mttkrp_coo3(I, J, Kd, ti, tj, tk, tv, Bt,
                                                                 Ct, A, ws))
        jobs["mttkrp_csf"] = (532_669_912, lambda: K.mttkrp_csf(I, J, Kd, c0, p1, c1, p2, c2, tv,
                                                                Bt, Ct, A, ws))

    if (want("coo") or want("hashx") or want("hashx_wdef") or want("csr_d1")
            or want("hashx_map") or want("hashx_wdef_map")):
        d1()
    if (want("csr") or want("coo_st") or want("ell") or want("csr_vec") or want("csr_merge") or want("csr_warp")
            or want("spmm4") or want("spmm16") or want("spmm32")):
        d2()
    if want("dia"):
        d3()
    if want("add"):
        d4()
    if want("mttkrp_coo") or want("mttkrp_csf"):
        d5()
    for name, (b, fn) in jobs.items():
        if only and name not in only:
            continue
        for _ in range(args.reps):
            K.l2_flush(flush)
            fn()
        torch.cuda.synchronize()
        if args.no_table:
            continue
        res = []
        for flushed in (True, False):
            ts = []
            for _ in range(20):
                if flushed:
                    K.l2_flush(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = float(np.mean(ts))
            res.append(f"{t * 1e3:9.2f} us {b / t / 1e6:8.1f} GB/s")
        print(f"{name:12s} flushed: {res[0]}   L2-warm: {res[1]}", flush=True)


if __name__ == "__main__":
    main()
