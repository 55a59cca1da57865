#!/usr/bin/env python
"""Benchmark of the B200 sparse level-format hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--no-formats]

Headline workload (BASELINE.json configs[1], the config its metric is quoted
on): "ELL vs CSR SpMV, fp64, 27-point stencil on a 64^3 grid".  One step =
one CSR SpMV and one ELL SpMV of the same matrix, each preceded by an L2
flush (the 87 MB working set would otherwise sit in the 126 MB L2).
value = compulsory bytes of both SpMVs / their summed kernel time (GB/s,
CUDA events on the launching stream, max over ranks).  The other BASELINE
configs (COO, DIA, A+B, MTTKRP COO-3/CSF) and the hashed-x SpMV are measured
in the same run and reported under "formats" (unless --no-formats).

Multi-GPU (torchrun, N ranks): weak scaling — rank r owns the z-slab
[64r, 64(r+1)) of a 64 x 64 x 64N stencil grid (an nnz-balanced row block of
the global matrix), x is replicated by one NCCL broadcast before timing, and
there is no collective inside the timed region.

--impl reference: the reference's CPU implementation of the same step on the
host cores.  The reference (`sparselevels`) is pure Python and is not present
on the GPU box, so this arm runs the C restatement of it (oracle/, bit-identical
to the reference on the golden vectors), multithreaded across all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMV effective HBM GB/s (% of peak) per format; MTTKRP nnz/s"
E2E_STREAMS = 4                         # e2e pipelining depth (tools/e2e_probe.py: 4 beats 3, 6 no better)
WORKLOAD = "ELL vs CSR SpMV fp64, 27-point stencil 64^3 (BASELINE configs[1])"
G = 64


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def l2_calib():
    """Measured L2 -> SM ceilings (tools/calib_l2.py on this pool's B200)."""
    p = ROOT / "profiles" / "l2_calib.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return {}


def ncu_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# algorithmic (compulsory) bytes per launch, SURVEY.md §8(d)

def bytes_csr(nrows, nnz):
    return 4 * (nrows + 1) + 12 * nnz + 8 * nrows + 8 * nrows   # pos, crd+vals, x, y


def bytes_ell(nrows, nslots):
    return 12 * nslots * nrows + 16 * nrows


def bytes_coo(nrows, ncols, nnz):
    return 16 * nnz + 8 * ncols + 8 * nrows


def bytes_dia(nrows, ncols, offsets):
    in_range = sum(max(0, min(nrows, ncols - o) - max(0, -o)) for o in offsets)
    return 8 * in_range + 8 * ncols + 8 * nrows + 4 * len(offsets)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# timing

class KernelTimer:
    """Per-launch CUDA-event timing with an L2 flush before every launch."""

    def __init__(self, torch, K, flush_bytes):
        self.torch = torch
        self.K = K
        self.flush = torch.empty(int(flush_bytes), dtype=torch.uint8, device="cuda")
        # "write+read" (default): the write sweep is followed by a read sweep of
        # another 2x-L2 buffer, so the timed kernel starts with a cold AND clean
        # L2 (no write-backs of the flush's dirty lines charged to it);
        # SL_BENCH_FLUSH=write keeps only the write sweep
        self.mode = os.environ.get("SL_BENCH_FLUSH", "write+read")
        self.rbuf = (torch.zeros(int(flush_bytes), dtype=torch.uint8, device="cuda")
                     if self.mode == "write+read" else None)
        self.sink = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.launches = 0        # timed kernel launches (inside the event brackets)
        self.flush_launches = 0  # L2 sweeps between them (ours too, outside the brackets)

    def _flush(self):
        self.K.l2_flush(self.flush)
        if self.rbuf is not None:
            self.K.l2_read(self.rbuf, self.sink)

    def run(self, fns, steps, warmup):
        """fns: {name: callable}; returns {name: [ms per step]}"""
        torch, K = self.torch, self.K
        for _ in range(warmup):
            for fn in fns.values():
                self._flush()
                fn()
        torch.cuda.synchronize()
        evs = {n: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)] for n in fns}
        for s in range(steps):
            for n, fn in fns.items():
                self._flush()
                e0, e1 = evs[n][s]
                e0.record()
                fn()
                e1.record()
                self.launches += 1
                self.flush_launches += 2 if self.rbuf is not None else 1
        torch.cuda.synchronize()
        return {n: [e0.elapsed_time(e1) for e0, e1 in evs[n]] for n in fns}


def l2_bytes(torch):
    try:
        return int(torch.cuda.get_device_properties(0).L2_cache_size)
    except Exception:
        return 126 * 2 ** 20


# ---------------------------------------------------------------------------
# our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1804_10112_b200 import dist as D
    from paper_1804_10112_b200 import formats as F
    from paper_1804_10112_b200 import kernels as K
    from paper_1804_10112_b200 import workloads as wl
    from paper_1804_10112_b200.engine import evaluate

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    peak, peak_src = measured_peak()
    traffic_db = ncu_traffic()

    # ---- headline instance: this rank's z-slab of a 64 x 64 x 64*world grid
    st = wl.stencil27(g=G, gz=G * world, z0=G * rank, z1=G * (rank + 1))
    nrows, ncols, nnz = st["nrows"], st["ncols"], len(st["crd"])
    ell = wl.csr_to_ell(st["pos"], st["crd"], st["vals"], nrows)
    S = ell["nslots"]
    pos, crd, vals = (torch.as_tensor(a, device=dev) for a in (st["pos"], st["crd"], st["vals"]))
    ecrd, evals = torch.as_tensor(ell["crd"], device=dev), torch.as_tensor(ell["vals"], device=dev)
    x = torch.as_tensor(st["x"], device=dev)
    if world > 1:
        D.replicate(x, src=0)            # x replicated once (NCCL broadcast), outside timing
    y1 = torch.empty(nrows, dtype=torch.float64, device=dev)
    y2 = torch.empty(nrows, dtype=torch.float64, device=dev)
    b_csr, b_ell = bytes_csr(nrows, nnz), bytes_ell(nrows, S)

    timer = KernelTimer(torch, K, 2 * l2_bytes(torch))
    fns = {"csr": lambda: K.spmv_csr(nrows, ncols, pos, crd, vals, x, y1),
           "ell": lambda: K.spmv_ell(nrows, ncols, S, ecrd, evals, x, y2)}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        times = timer.run(fns, args.steps, args.warmup)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_csr, t_ell = float(np.sum(times["csr"])), float(np.sum(times["ell"]))
    t_total = D.max_over_ranks(t_csr + t_ell, dev)          # ms over K steps, max over ranks
    bytes_all = D.sum_over_ranks(float(b_csr + b_ell) * args.steps, dev)
    value = bytes_all / (t_total * 1e-3) / 1e9
    launches = timer.launches                                # SpMV launches inside the events

    # roofline: dominant kernel of the step
    avg = {"csr": t_csr / args.steps, "ell": t_ell / args.steps}
    dom = max(avg, key=avg.get)
    dom_bytes = b_csr if dom == "csr" else b_ell
    achieved = dom_bytes / (avg[dom] * 1e-3) / 1e9
    kname = {"csr": "spmv_csr_handoff_kernel", "ell": "spmv_ell_kernel"}[dom]
    traffic = traffic_db.get(kname)

    # ---- e2e through the public API: x from pinned host memory each step,
    # the matrix resident on the device (like weights), y read back.  Steps
    # rotate over E2E_STREAMS streams (each with its own pinned x / y buffers),
    # so step k+1's host->device copy overlaps step k's kernel and device->host copy —
    # a serving loop's pipelining; every step still moves its own x in and y out.
    A_st = F.csr_storage(pos, crd, vals, (nrows, ncols), device=dev)
    ns = E2E_STREAMS
    x_hosts = [torch.as_tensor(st["x"]).pin_memory() for _ in range(ns)]
    xs = [F.dense_storage(xh, device=None) for xh in x_hosts]
    y_hosts = [torch.empty(nrows, dtype=torch.float64).pin_memory() for _ in range(ns)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(ns)]
    expr = "y(i) = A(i,j) * x(j)"

    def e2e_step(k):
        with torch.cuda.stream(streams[k % ns]):
            y_dev = evaluate(expr, {"A": A_st, "x": xs[k % ns]}).vals
            y_hosts[k % ns].copy_(y_dev, non_blocking=True)

    for k in range(max(args.warmup, 3)):
        e2e_step(k)
    torch.cuda.synchronize()
    e2e_steps = max(10, min(args.steps, 200))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        e2e_step(k)
    torch.cuda.synchronize()
    t_e2e = D.max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev)
    e2e_val = D.sum_over_ranks(float(b_csr), dev) / t_e2e / 1e9

    out = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_total / args.steps, 6),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded numpy; BASELINE configs have no public dataset)",
        "config": {"workload": WORKLOAD, "grid": f"{G}x{G}x{G * world}",
                   "rows_per_gpu": nrows, "nnz_per_gpu": nnz, "ell_slots": S,
                   "step": "CSR SpMV + ELL SpMV, each after an L2 flush",
                   "l2": (f"flushed before every launch ({2 * l2_bytes(torch) >> 20} MiB write sweep"
               + (f" + {2 * l2_bytes(torch) >> 20} MiB read sweep: cold and clean)"
                  if timer.mode == "write+read" else ")")),
                   "parallelism": f"row-block shards x{world}, x replicated (NCCL broadcast)"},
        "pct_of_peak": round(100.0 * value / (peak * world), 2),
        "per_kernel_ms": {k: round(v, 6) for k, v in avg.items()},
        "per_kernel_gbs": {"csr": round(b_csr / (avg["csr"] * 1e-3) / 1e9, 1),
                           "ell": round(b_ell / (avg["ell"] * 1e-3) / 1e9, 1)},
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "algorithmic_bytes": dom_bytes,
                     "traffic": traffic},
        "e2e": {"value": round(e2e_val, 3), "unit": "GB/s",
                "h2d_bytes_per_step": int(x_hosts[0].numel() * 8),
                "d2h_bytes_per_step": int(nrows * 8),
                "ms_per_step": round(t_e2e * 1e3, 4),
                "path": "evaluate('y(i) = A(i,j) * x(j)') CSR, pinned host x in, y out every "
                        f"step; matrix resident in HBM; steps rotate over {ns} streams"},
        "gpu_launches": launches,
        "gpu_launches_note": (f"{launches} SpMV kernel launches inside the timed events "
                              f"(CSR + ELL per step); plus {timer.flush_launches} L2-sweep "
                              "launches between them"),
        "clocks": clk.summary(),
    }

    # ---- optional all-gather of the y row blocks (N > 1), timed on its own:
    # the one data-path collective the north star allows after compute
    if world > 1:
        bounds = [nrows * p for p in range(world + 1)]
        for _ in range(3):
            D.gather_row_blocks(y1, bounds)
        torch.cuda.synchronize()
        dist.barrier()
        reps = 20
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(reps):
            yfull = D.gather_row_blocks(y1, bounds)
        g1.record()
        torch.cuda.synchronize()
        t_ag = D.max_over_ranks(g0.elapsed_time(g1) / reps, dev)
        out["y_allgather"] = {"ms": round(t_ag, 5), "bytes_per_rank_out": nrows * 8,
                              "full_y_bytes": int(yfull.numel() * 8),
                              "GB/s_per_rank_in": round(yfull.numel() * 8 / (t_ag * 1e-3) / 1e9, 1),
                              "note": "torch.distributed all_gather of padded y blocks "
                                      "(NCCL); not part of `value`"}

    # ---- MTTKRP across ranks (N > 1, BASELINE configs[4]): nnz-balanced slice
    # blocks of the one D5 tensor (strong scaling: total work fixed), factors
    # replicated by broadcast, each rank writes its disjoint block of A rows
    if world > 1 and not args.no_formats:
        mt = wl.mttkrp()
        I, J, Kd, R = mt["I"], mt["J"], mt["K"], mt["R"]
        sb = D.slice_blocks_coo3(mt["i"], I, world)
        s0, s1 = int(sb[rank]), int(sb[rank + 1])
        ii, jj, kk, vv = D.shard_coo3(mt["i"], mt["j"], mt["k"], mt["vals"], s0, s1)
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
        ti, tj, tk, tv = T(ii), T(jj), T(kk), T(vv)
        Bt = torch.empty((J, R), dtype=torch.float64, device=dev)
        Ct = torch.empty((Kd, R), dtype=torch.float64, device=dev)
        if rank == 0:
            Bt.copy_(torch.as_tensor(mt["B"]).reshape(J, R))
            Ct.copy_(torch.as_tensor(mt["C"]).reshape(Kd, R))
        D.replicate(Bt, src=0)
        D.replicate(Ct, src=0)
        At = torch.empty((s1 - s0, R), dtype=torch.float64, device=dev)
        ws = torch.empty(int(K.L().sl_mttkrp_workspace_bytes(len(ii), R)), dtype=torch.uint8,
                         device=dev)
        nloc = len(ii)
        del mt
        dist.barrier()
        tm = timer.run({"mttkrp": lambda: K.mttkrp_coo3(s1 - s0, J, Kd, ti, tj, tk, tv, Bt, Ct,
                                                       At, ws=ws)}, 10, 3)
        t_mt = D.max_over_ranks(float(np.mean(tm["mttkrp"])), dev)      # ms
        nnz_all = D.sum_over_ranks(float(nloc), dev)
        out["mttkrp_coo3_sharded"] = {
            "ms": round(t_mt, 5), "nnz/s": round(nnz_all / (t_mt * 1e-3), 1),
            "nnz*R/s": round(nnz_all * R / (t_mt * 1e-3), 1),
            "GFLOP/s": round(3 * nnz_all * R / (t_mt * 1e-3) / 1e9, 1),
            "nnz_per_rank_max_over_mean": round(
                D.max_over_ranks(float(nloc), dev) / (nnz_all / world), 4),
            "scaling": "strong", "note": "slice blocks balanced by nnz; B, C broadcast; "
                                         "max over ranks of the mean launch time"}

    # ---- CPU baseline (rank 0, N = 1): the oracle port on the host cores
    if rank == 0 and world == 1:
        out["cpu_baseline"] = cpu_baseline(st, ell, args)

    # ---- the other BASELINE configs, same run (N = 1)
    if world == 1 and not args.no_formats:
        out["formats"] = run_formats(torch, K, wl, dev, timer, peak, max(5, min(args.steps, 30)))
    return out


def cpu_baseline(st, ell, args, budget_s=10.0):
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # test infrastructure: CPU baseline leg only

    thr = oracle.num_threads()
    nrows = st["nrows"]
    b = bytes_csr(nrows, len(st["crd"])) + bytes_ell(nrows, ell["nslots"])
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s and n < 200:
        oracle.spmv_csr(nrows, st["pos"], st["crd"], st["vals"], st["x"], threads=thr)
        oracle.spmv_ell(nrows, ell["nslots"], ell["crd"], ell["vals"], st["x"], threads=thr)
        n += 1
    dt = (time.perf_counter() - t0) / n
    return {"value": round(b / dt / 1e9, 3), "unit": "GB/s", "cores": thr, "kind": "port",
            "sample": f"{n} steps of CSR+ELL SpMV on the full 64^3 stencil, "
                      f"{dt * 1e3:.2f} ms/step, C restatement of the reference (oracle/)",
            "host_cpu_count": os.cpu_count()}


def run_formats(torch, K, wl, dev, timer, peak, steps):
    """Kernel-only numbers for the other BASELINE configs (same timing rules)."""
    res = {}
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731

    d = wl.coo_spmv()
    n, m, nnz = d["nrows"], d["ncols"], len(d["rows"])
    r, c, v, x = T(d["rows"]), T(d["cols"]), T(d["vals"]), T(d["x"])
    y = torch.empty(n, dtype=torch.float64, device=dev)
    pos = T(wl.coo_to_csr_pos(d["rows"], n))
    h = wl.hash_vector()
    hc, hv = T(h["crd"]), T(h["vals"])
    hws = torch.empty(int(K.L().sl_spmv_csr_hashx_map_workspace_bytes(m, h["width"])),
                      dtype=torch.uint8, device=dev)
    tt = timer.run({"coo": lambda: K.spmv_coo(n, m, r, c, v, x, y),
                    "csr_hashx": lambda: K.spmv_csr_hashx(n, pos, c, v, h["width"], hc, hv, y),
                    "csr_hashx_map": lambda: K.spmv_csr_hashx(n, pos, c, v, h["width"], hc, hv, y,
                                                              n=m, ws=hws)},
                   steps, 3)
    b = bytes_coo(n, m, nnz)
    t = float(np.mean(tt["coo"]))
    g8 = l2_calib().get("gather8_20M_G_per_s") or l2_calib().get("gather8_G_per_s")
    res["coo_spmv_D1"] = {"ms": round(t, 5), "GB/s": round(b / t / 1e6, 1),
                          "frac": round(b / t / 1e6 / peak, 4), "nnz/s": round(nnz / t * 1e3, 1),
                          "bytes": b,
                          "gather_ceiling": {"x_gathers": nnz, "peak_G_per_s": g8,
                                             "floor_ms": round(nnz / g8 / 1e6, 5) if g8 else None,
                                             "note": "random 8-B x gathers at the throughput measured over 20M gathers (tools/calib_l2.py); a floor for the gathers alone, overlappable with the 35 MB stream"}}
    bh = 4 * (n + 1) + 12 * nnz + 8 * n + 12 * h["width"]
    t = float(np.mean(tt["csr_hashx"]))
    res["csr_hashx_H1"] = {"ms": round(t, 5), "GB/s": round(bh / t / 1e6, 1),
                           "locates/s": round(nnz / t * 1e3, 1), "bytes": bh,
                           "path": "per-nonzero warp-cooperative probing"}
    t = float(np.mean(tt["csr_hashx_map"]))
    res["csr_hashx_map_H1"] = {"ms": round(t, 5), "GB/s": round(bh / t / 1e6, 1),
                               "locates/s": round(nnz / t * 1e3, 1), "bytes": bh,
                               "path": "slot map (one locate per coordinate) + CSR SpMV"}
    # format conversion (formats.convert): the COO -> CSR identity copy, and
    # the structural row pointer alone; the paper's "convert, then CSR SpMV"
    # alternative to COO SpMV costs convert + csr_spmv_D1.
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    tt = timer.run({"conv": lambda: K.coo_to_csr(n, r, c, v, sync=False),
                    "rowptr": lambda: K.coo_rowptr(n, r, rp),
                    "csr": lambda: K.spmv_csr(n, m, pos, c, v, x, y)}, steps, 3)
    bc = 16 * nnz + 4 * (n + 1) + 12 * nnz
    t = float(np.mean(tt["conv"]))
    res["convert_coo_to_csr_D1"] = {"ms": round(t, 5), "GB/s": round(bc / t / 1e6, 1),
                                    "frac": round(bc / t / 1e6 / peak, 4), "bytes": bc}
    br = 4 * nnz + 4 * (n + 1)
    t = float(np.mean(tt["rowptr"]))
    res["coo_rowptr_D1"] = {"ms": round(t, 5), "GB/s": round(br / t / 1e6, 1), "bytes": br}
    bs = bytes_csr(n, nnz)
    t = float(np.mean(tt["csr"]))
    res["csr_spmv_D1"] = {"ms": round(t, 5), "GB/s": round(bs / t / 1e6, 1),
                          "frac": round(bs / t / 1e6 / peak, 4), "bytes": bs}
    # the paper's end-to-end question (Fig. 13): COO SpMV on unconverted
    # coordinates vs converting to CSR first (exact identity copy) and then CSR SpMV
    res["coo_vs_convert_then_csr_D1"] = {
        "coo_spmv_ms": res["coo_spmv_D1"]["ms"],
        "convert_plus_csr_ms": round(res["convert_coo_to_csr_D1"]["ms"] + t, 5),
        "rowptr_only_plus_csr_ms": round(res["coo_rowptr_D1"]["ms"] + t, 5)}
    del r, c, v, x, y, pos, rp

    # widened patterns on the headline stencil: SpMM with
    # K = 16 dense columns, and CSR x sparse-vector x holding half the coordinates
    st = wl.stencil27()
    n, nnz = st["nrows"], len(st["crd"])
    sp, sc, sv = T(st["pos"]), T(st["crd"]), T(st["vals"])
    Kc = 16
    rng = np.random.default_rng(5)
    Xd = T(rng.uniform(-1, 1, (n, Kc)))
    Yd = torch.empty((n, Kc), dtype=torch.float64, device=dev)
    keep = np.sort(rng.choice(n, n // 2, replace=False)).astype(np.int32)
    xk, xkv = T(keep), T(rng.uniform(-1, 1, len(keep)))
    ys = torch.empty(n, dtype=torch.float64, device=dev)
    sws = torch.empty(int(K.L().sl_spmv_csr_spx_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    tt = timer.run({"spmm": lambda: K.spmm_csr(n, n, sp, sc, sv, Xd, Yd),
                    "spx": lambda: K.spmv_csr_spx(n, n, sp, sc, sv, xk, xkv, ys, sws)}, steps, 3)
    b = 4 * (n + 1) + 12 * nnz + 16 * n * Kc
    t = float(np.mean(tt["spmm"]))
    res["spmm_csr_stencil_K16"] = {"ms": round(t, 5), "GB/s": round(b / t / 1e6, 1),
                                   "frac": round(b / t / 1e6 / peak, 4), "bytes": b,
                                   "GFLOP/s": round(2 * nnz * Kc / t / 1e6, 1)}
    b = 4 * (n + 1) + 12 * nnz + 12 * len(keep) + 8 * n
    t = float(np.mean(tt["spx"]))
    res["spmv_csr_spx_stencil"] = {"ms": round(t, 5), "GB/s": round(b / t / 1e6, 1),
                                   "frac": round(b / t / 1e6 / peak, 4), "bytes": b,
                                   "x_nnz": int(len(keep))}
    del sp, sc, sv, Xd, Yd, xk, xkv, ys, sws

    g = wl.dia7()
    n = g["nrows"]
    gv, gx = T(g["vals"]), T(g["x"])
    y = torch.empty(n, dtype=torch.float64, device=dev)
    tt = timer.run({"dia": lambda: K.spmv_dia(n, n, g["offsets"], gv, gx, y)}, steps, 3)
    b = bytes_dia(n, n, g["offsets"].tolist())
    t = float(np.mean(tt["dia"]))
    res["dia_spmv_D3"] = {"ms": round(t, 5), "GB/s": round(b / t / 1e6, 1),
                          "frac": round(b / t / 1e6 / peak, 4), "bytes": b}
    del gv, gx, y

    a = wl.add_ab()
    n = a["nrows"]
    ap, ac, av = T(a["a_pos"]), T(a["a_crd"]), T(a["a_vals"])
    br, bc, bv = T(a["b_rows"]), T(a["b_cols"]), T(a["b_vals"])
    out = {}

    def add():
        out["c"] = K.add_csr(n, ap, ac, av, bc, bv, b_rows=br, sync=False)

    tt = timer.run({"add": add}, steps, 3)
    nnz_c = int(out["c"][0][n].item())
    b = 4 * (n + 1) + 12 * len(a["a_crd"]) + 16 * len(a["b_cols"]) + 4 * (n + 1) + 12 * nnz_c
    t = float(np.mean(tt["add"]))
    res["add_csr_coo_D4"] = {"ms": round(t, 5), "GB/s": round(b / t / 1e6, 1),
                             "frac": round(b / t / 1e6 / peak, 4), "nnz_c": nnz_c, "bytes": b,
                             "input nnz/s": round((len(a["a_crd"]) + len(a["b_cols"])) / t * 1e3, 1)}
    del ap, ac, av, br, bc, bv, out

    mt = wl.mttkrp()
    csf = wl.coo3_to_csf(mt["i"], mt["j"], mt["k"], None)
    I, J, Kd, R = mt["I"], mt["J"], mt["K"], mt["R"]
    nnz = len(mt["i"])
    ti, tj, tk, tv = T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"])
    Bt, Ct = T(mt["B"]), T(mt["C"])
    c0, p1, c1, p2, c2 = (T(csf[k]) for k in ("crd0", "pos1", "crd1", "pos2", "crd2"))
    A = torch.empty((I, R), dtype=torch.float64, device=dev)
    ws = torch.empty(int(K.L().sl_mttkrp_workspace_bytes(nnz, R)), dtype=torch.uint8, device=dev)
    tt = timer.run({"coo3": lambda: K.mttkrp_coo3(I, J, Kd, ti, tj, tk, tv, Bt, Ct, A, ws),
                    "csf": lambda: K.mttkrp_csf(I, J, Kd, c0, p1, c1, p2, c2, tv, Bt, Ct, A, ws)},
                   max(3, steps // 3), 2)
    bf = 8 * (J * R + Kd * R + I * R)
    b_coo = 20 * nnz + bf
    n1 = len(csf["crd1"])
    b_csf = 8 + 4 * len(csf["crd0"]) + 4 * (len(csf["crd0"]) + 1) + 4 * n1 + 4 * (n1 + 1) + 12 * nnz + bf
    # L2 -> SM bytes the loop nest must move at minimum: a C row per nonzero and
    # a B row per (i, j) fiber (factors are L2-resident, L1 far smaller), plus
    # the streamed tensor and the A rows — the resource that bounds MTTKRP.
    l2c = l2_calib()
    l2_peak = l2c.get("gather256_GBs")
    l2_rows = 8 * R * (nnz + n1) + 8 * I * R
    for name, b, key in (("mttkrp_coo3_D5", b_coo, "coo3"), ("mttkrp_csf_D5", b_csf, "csf")):
        t = float(np.mean(tt[key]))
        l2b = l2_rows + (b - bf)
        res[name] = {"ms": round(t, 4), "nnz/s": round(nnz / t * 1e3, 1),
                     "nnz*R/s": round(nnz * R / t * 1e3, 1), "GB/s": round(b / t / 1e6, 1),
                     "frac": round(b / t / 1e6 / peak, 4), "GFLOP/s": round(3 * nnz * R / t / 1e6, 1),
                     "bytes": b,
                     "l2_roofline": {"bound": "l2 (factor-row gathers)", "bytes": l2b,
                                     "achieved_GBs": round(l2b / t / 1e6, 1),
                                     "peak_GBs": l2_peak,
                                     "peak_source": "profiles/l2_calib.json gather256_GBs "
                                                    "(tools/calib_l2.py, 256-B random rows)",
                                     "frac": round(l2b / t / 1e6 / l2_peak, 4) if l2_peak else None}}

    # the paper's other kernels on the same tensor: TTV into a
    # CSR-over-fibers output (a per-fibre SpMV + the fibre row pointer) and
    # INNERPROD of the COO-3 tensor with itself (intersection at every level)
    vt = T(np.random.default_rng(3).uniform(-1.0, 1.0, Kd))
    zi, zj, zk, zv = ti.clone(), tj.clone(), tk.clone(), tv.clone()
    tt = timer.run({"ttv": lambda: K.ttv_csf(I, J, Kd, c0, p1, c1, p2, c2, tv, vt, out="csr"),
                    "inner": lambda: K.inner_coo3(I, J, Kd, (ti, tj, tk, tv), (zi, zj, zk, zv))},
                   max(3, steps // 3), 2)
    t = float(np.mean(tt["ttv"]))
    b_ttv = (4 * (len(csf["crd0"]) + 1) + 4 * len(csf["crd0"]) + 4 * (n1 + 1) + 12 * nnz + 8 * Kd
             + 4 * (I + 1) + 12 * n1)
    res["ttv_csf_csr_out_D5"] = {"ms": round(t, 4), "GB/s": round(b_ttv / t / 1e6, 1),
                                 "frac": round(b_ttv / t / 1e6 / peak, 4), "bytes": b_ttv,
                                 "nnz/s": round(nnz / t * 1e3, 1), "fibers": n1}
    t = float(np.mean(tt["inner"]))
    b_in = 2 * 20 * nnz
    res["innerprod_coo3_D5"] = {"ms": round(t, 4), "GB/s": round(b_in / t / 1e6, 1),
                                "frac": round(b_in / t / 1e6 / peak, 4), "bytes": b_in,
                                "nnz/s": round(nnz / t * 1e3, 1)}
    return res


# ---------------------------------------------------------------------------
# reference arm

def run_reference(args, rank, world):
    if rank != 0:
        return None
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # the reference's CPU path (C restatement; see module docstring)

    from paper_1804_10112_b200 import workloads as wl

    st = wl.stencil27(g=G, gz=G * world, z0=0, z1=G * world)
    ell = wl.csr_to_ell(st["pos"], st["crd"], st["vals"], st["nrows"])
    # every host thread this process may run on (torchrun exports
    # OMP_NUM_THREADS=1, which would otherwise pin the reference arm to 1 core)
    thr = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nrows = st["nrows"]
    b = bytes_csr(nrows, len(st["crd"])) + bytes_ell(nrows, ell["nslots"])
    for _ in range(args.warmup):
        oracle.spmv_csr(nrows, st["pos"], st["crd"], st["vals"], st["x"], threads=thr)
        oracle.spmv_ell(nrows, ell["nslots"], ell["crd"], ell["vals"], st["x"], threads=thr)
    steps = min(args.steps, 200)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.spmv_csr(nrows, st["pos"], st["crd"], st["vals"], st["x"], threads=thr)
        oracle.spmv_ell(nrows, ell["nslots"], ell["crd"], ell["vals"], st["x"], threads=thr)
    dt = (time.perf_counter() - t0) / steps
    value = b / dt / 1e9
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "grid": f"{G}x{G}x{G * world}",
                   "step": "CSR SpMV + ELL SpMV (host)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": thr, "kind": "port",
                         "sample": f"{steps} full steps; C restatement of the reference "
                                   "(the Python reference is absent on the GPU box)"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-formats", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch
    import torch.distributed as dist

    # one rank per GPU; SL_BENCH_BACKEND=gloo (with ranks folded onto the
    # visible GPUs) only smoke-tests the multi-rank code path on a 1-GPU box —
    # its numbers are not measurements
    local_rank = local_rank % max(1, torch.cuda.device_count())
    backend = os.environ.get("SL_BENCH_BACKEND", "nccl")
    if world > 1:
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    from paper_1804_10112_b200 import _lib

    _lib.load()   # fail loudly if the kernel library is missing
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
