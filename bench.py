#!/usr/bin/env python
"""Benchmark of the B200 sparse level-format hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--no-formats]

Headline workload (BASELINE.json configs[1], the config its metric is quoted
on): "ELL vs CSR SpMV, fp64, 27-point stencil on a 64^3 grid".  One step =
one CSR SpMV and one ELL SpMV of the same matrix.  value = compulsory bytes
of both SpMVs / their kernel time (GB/s, CUDA events on the launching
stream, max over ranks).

L2 protocol: inputs larger than L2.  Every operand (matrix arrays, x, y) is
held in enough device copies that the copies a kernel did not touch in its
last launch exceed the 126 MB L2 eightfold; launch s reads copy s mod n, so
each launch finds its operands cold (ncu with --cache-control none over the
rotation: 84.5 MB of DRAM reads per CSR launch against 85.4 MB algorithmic
reads — profiles/r2_ncu_rotation.txt; with a 1.5x margin L2 still served
~3 MB of high-reuse lines, x among them, and the kernels timed ~5% faster).
The K launches of a kernel are captured once into a CUDA graph and replayed
back to back inside one event pair: a per-launch event bracket costs ~6 us on
this part even around an empty kernel (tools/calib_overhead.cu,
profiles/r2_calib_overhead.txt), and issuing from Python leaves the GPU
waiting on the host's ~15 us per ctypes call.
SL_BENCH_L2=flush selects the round-1 protocol instead (a 2x-L2 write sweep
and read sweep before every launch, one event pair per launch).

The other BASELINE configs (COO, DIA, A+B, MTTKRP COO-3/CSF) and the hashed-x
SpMV are measured in the same run under "formats" (unless --no-formats), each
with its own e2e (through `evaluate`, host buffers in and out) and its CPU
baseline (the oracle port on the host cores).

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
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMV effective HBM GB/s (% of peak) per format; MTTKRP nnz/s"
E2E_STREAMS = int(os.environ.get("SL_E2E_STREAMS", "4"))   # e2e pipelining depth (tools/e2e_probe.py: 4 beats 3, 6 no better)
WORKLOAD = "ELL vs CSR SpMV fp64, 27-point stencil 64^3 (BASELINE configs[1])"
G = 64
L2_MARGIN = float(os.environ.get("SL_BENCH_L2_MARGIN", "8"))   # rotated copies exceed L2 by this factor


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


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def headline_config(world, rows_per_gpu, nnz_per_gpu, slots):
    """The workload, identical in both arms (the measurement protocol is
    reported separately under "timing")."""
    return {"workload": WORKLOAD, "grid": f"{G}x{G}x{G * world}", "rows_per_gpu": rows_per_gpu,
            "nnz_per_gpu": nnz_per_gpu, "ell_slots": slots,
            "step": "CSR SpMV + ELL SpMV of the same matrix"}


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
# clocks: NVML polled every ~0.5 ms from a thread, samples tagged with the
# timed region they fall in (nvidia-smi -lms cannot resolve a ~1 ms region)

class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.samples = []            # (region or None, sm_mhz, reasons bitmask)
        self.region = None
        self.stop = threading.Event()
        self.max_mhz = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _poll(self):
        nv, h = self.nv, self.h
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((self.region, float(sm), int(rs)))
            except Exception:
                pass
            time.sleep(0.0005)

    def timed(self, name):
        sampler = self

        class _R:
            def __enter__(self_):
                sampler.region = name

            def __exit__(self_, *a):
                sampler.region = None
        return _R()

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self, region=None):
        sel = [s for s in self.samples if s[0] is not None and (region is None or s[0] == region)]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = set()
        for _, _, rs in sel:
            for bit, nm in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median([s[1] for s in sel])), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sel)}


# ---------------------------------------------------------------------------
# timing

def copies_for(nbytes, l2):
    """Device copies a kernel rotates through so that the copies it did not
    touch in its last launch exceed L2 by L2_MARGIN."""
    return max(2, 1 + math.ceil(L2_MARGIN * l2 / max(nbytes, 1)))


class KernelTimer:
    """Times K launches of each kernel back to back in one CUDA-event pair on
    the launching (current) stream, rotating over device copies of its
    operands whose total exceeds L2 (or, SL_BENCH_L2=flush, the round-1
    per-launch flush protocol)."""

    def __init__(self, torch, K, l2):
        self.torch = torch
        self.K = K
        self.l2 = l2
        self.mode = os.environ.get("SL_BENCH_L2", "rotate")
        if self.mode == "flush":
            self.flush = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")
            self.rbuf = torch.zeros(2 * l2, dtype=torch.uint8, device="cuda")
            self.sink = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.launches = 0            # timed kernel launches (inside the event brackets)
        self.graphs = os.environ.get("SL_BENCH_GRAPH", "1") != "0"
        self.method = {}             # kernel -> "graph" | "stream"

    def describe(self):
        if self.mode == "flush":
            return (f"flushed before every launch ({2 * self.l2 >> 20} MiB write sweep + "
                    f"{2 * self.l2 >> 20} MiB read sweep), one event pair per launch")
        return (f"inputs larger than L2: each kernel rotates over device copies of all its "
                f"operands totalling >= {L2_MARGIN}x the {self.l2 >> 20} MiB L2 beyond the copy "
                f"in use; its K launches back to back in one event pair (no flush), submitted "
                f"as one CUDA graph replay")

    def run(self, fns, steps, warmup, capture=True):
        """fns: {name: [callable per operand copy]}; returns {name: ms per launch}.
        capture=False: the callables read the device between launches (data-
        dependent output sizes), so no graph capture is attempted."""
        torch = self.torch
        out = {}
        for name, copies in fns.items():
            nc = len(copies)
            for w in range(max(warmup, nc)):
                copies[w % nc]()
            torch.cuda.synchronize()
            if self.mode == "flush":
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(steps)]
                for s in range(steps):
                    self.K.l2_flush(self.flush)
                    self.K.l2_read(self.rbuf, self.sink)
                    evs[s][0].record()
                    copies[s % nc]()
                    evs[s][1].record()
                torch.cuda.synchronize()
                out[name] = float(np.mean([a.elapsed_time(b) for a, b in evs]))
            else:
                out[name] = self._rotate(name, copies, steps, capture)
            self.launches += steps
        return out

    def _rotate(self, name, copies, steps, capture=True):
        """K launches rotating over the copies, back to back in one event pair.
        They are captured once into a CUDA graph and the graph is replayed
        inside the events, so the host's per-call cost (ctypes marshalling,
        ~10-20 us) cannot starve a ~15 us kernel; if a kernel's wrapper cannot
        be captured, the launches are issued directly on the stream."""
        torch = self.torch
        nc = len(copies)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g = None
        if self.graphs and capture:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for s in range(steps):
                        copies[s % nc]()
                g.replay()                      # warm replay (untimed)
                torch.cuda.synchronize()
            except Exception:
                g = None
                torch.cuda.synchronize()
        self.method[name] = "graph" if g is not None else "stream"
        e0.record()
        if g is not None:
            g.replay()
        else:
            for s in range(steps):
                copies[s % nc]()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps


def l2_bytes(torch):
    try:
        return int(torch.cuda.get_device_properties(0).L2_cache_size)
    except Exception:
        return 126 * 2 ** 20


def dev_copies(torch, arrays, n, dev):
    """n device copies of a tuple of host/device arrays (copy 0 may alias)."""
    base = [torch.as_tensor(a, device=dev) for a in arrays]
    return [tuple(t if c == 0 else t.clone() for t in base) for c in range(n)]


def e2e_loop(torch, steps, step_fn, warmup=3, batches=5):
    """Wall time per step of `step_fn(k)` (the public API, host buffers in and
    out, rotating over E2E_STREAMS streams), synchronised on both sides.
    Warm-up covers every pipeline slot twice (a slot's first use pays one-time
    stream / pinned-buffer set-up); the median of `batches` batches of `steps`
    steps is reported, so one host hiccup (a GC pause, another tenant of the
    box) cannot own a ~3 ms measurement."""
    for k in range(max(warmup, 2 * E2E_STREAMS)):
        step_fn(k)
    torch.cuda.synchronize()
    per = []
    for _ in range(batches):
        t0 = time.perf_counter()
        for k in range(steps):
            step_fn(k)
        torch.cuda.synchronize()
        per.append((time.perf_counter() - t0) / steps)
    return sorted(per)[len(per) // 2]


def time_cpu(fn, min_s=1.0, max_reps=10_000):
    """Wall time per call of a host function, repeated for at least min_s."""
    fn()
    n, t0 = 0, time.perf_counter()
    while True:
        fn()
        n += 1
        dt = time.perf_counter() - t0
        if dt >= min_s or n >= max_reps:
            return dt / n, n


# ---------------------------------------------------------------------------
# our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1804_10112_b200 import dist as D
    from paper_1804_10112_b200 import formats as F
    from paper_1804_10112_b200 import kernels as K
    from paper_1804_10112_b200 import workloads as wl
    from paper_1804_10112_b200.compiled import compile as compile_, compile_many
    from paper_1804_10112_b200.engine import evaluate

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    peak, peak_src = measured_peak()
    traffic_db = ncu_traffic()
    l2 = l2_bytes(torch)

    # ---- headline instance: this rank's z-slab of a 64 x 64 x 64*world grid
    st = wl.stencil27(g=G, gz=G * world, z0=G * rank, z1=G * (rank + 1))
    nrows, ncols, nnz = st["nrows"], st["ncols"], len(st["crd"])
    ell = wl.csr_to_ell(st["pos"], st["crd"], st["vals"], nrows)
    S = ell["nslots"]
    b_csr, b_ell = bytes_csr(nrows, nnz), bytes_ell(nrows, S)
    x0 = torch.as_tensor(st["x"], device=dev)
    if world > 1:
        D.replicate(x0, src=0)           # x replicated once (NCCL broadcast), outside timing
    xh = x0.cpu().numpy()
    ycsr = torch.empty(nrows, dtype=torch.float64)
    nc_csr, nc_ell = copies_for(b_csr, l2), copies_for(b_ell, l2)
    csr_ops = dev_copies(torch, (st["pos"], st["crd"], st["vals"], xh, ycsr), nc_csr, dev)
    ell_ops = dev_copies(torch, (ell["crd"], ell["vals"], xh, ycsr), nc_ell, dev)

    timer = KernelTimer(torch, K, l2)
    fns = {"csr": [lambda o=o: K.spmv_csr(nrows, ncols, o[0], o[1], o[2], o[3], o[4])
                   for o in csr_ops],
           "ell": [lambda o=o: K.spmv_ell(nrows, ncols, S, o[0], o[1], o[2], o[3])
                   for o in ell_ops]}
    out = {}
    with ClockSampler(local_rank) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with clk.timed("headline"):
            times = timer.run(fns, args.steps, args.warmup)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_csr, t_ell = times["csr"] * args.steps, times["ell"] * args.steps
        t_total = D.max_over_ranks(t_csr + t_ell, dev)          # ms over K steps, max over ranks
        bytes_all = D.sum_over_ranks(float(b_csr + b_ell) * args.steps, dev)
        value = bytes_all / (t_total * 1e-3) / 1e9
        launches = timer.launches                                # SpMV launches inside the events

        # roofline: dominant kernel of the step
        avg = {"csr": times["csr"], "ell": times["ell"]}
        dom = max(avg, key=avg.get)
        dom_bytes = b_csr if dom == "csr" else b_ell
        achieved = dom_bytes / (avg[dom] * 1e-3) / 1e9
        kname = {"csr": "spmv_csr_handoff_kernel", "ell": "spmv_ell_kernel"}[dom]
        traffic = traffic_db.get(kname)

        # ---- e2e through the public API: x from pinned host memory each step,
        # both matrices (CSR and ELL) resident on the device (like weights),
        # both y read back.  Steps rotate over E2E_STREAMS streams (own pinned
        # x / y buffers), so step k+1's host->device copy overlaps step k's
        # kernels and device->host copies — a serving loop's pipelining.
        pos, crd, vals = csr_ops[0][:3]
        A_csr = F.csr_storage(pos, crd, vals, (nrows, ncols), device=dev)
        A_ell = F.ell_storage(S, ell_ops[0][0], ell_ops[0][1], (nrows, ncols), device=dev)
        ns = E2E_STREAMS
        x_hosts = [torch.as_tensor(xh).pin_memory() for _ in range(ns)]
        xs = [F.dense_storage(t, device=None) for t in x_hosts]
        y_hosts = [(torch.empty(nrows, dtype=torch.float64).pin_memory(),
                    torch.empty(nrows, dtype=torch.float64).pin_memory()) for _ in range(ns)]
        streams = [torch.cuda.Stream(device=dev) for _ in range(ns)]
        expr = "y(i) = A(i,j) * x(j)"

        def eager_step(k):
            with torch.cuda.stream(streams[k % ns]):
                xd = xs[k % ns].to(dev, non_blocking=True)
                y1 = evaluate(expr, {"A": A_csr, "x": xd}).vals
                y2 = evaluate(expr, {"A": A_ell, "x": xd}).vals
                y_hosts[k % ns][0].copy_(y1, non_blocking=True)
                y_hosts[k % ns][1].copy_(y2, non_blocking=True)

        # the same step bound once with `compile_many`: per pipeline slot one
        # CUDA graph holding the x copy node (pinned host -> device), the two
        # SpMV kernels `evaluate` launches and the two y copy nodes (device ->
        # pinned host); a step is one graph launch on the slot's stream
        bound = [compile_many([(expr, {"A": A_csr, "x": xs[s]}, None),
                               (expr, {"A": A_ell, "x": xs[s]}, None)]) for s in range(ns)]

        def e2e_step(k):
            bound[k % ns](streams[k % ns])

        e2e_steps = max(50, min(args.steps, 200))
        if world > 1:
            dist.barrier()
        with clk.timed("e2e"):
            t_eager = D.max_over_ranks(e2e_loop(torch, e2e_steps, eager_step, max(args.warmup, 3)),
                                       dev)
            t_e2e = D.max_over_ranks(e2e_loop(torch, e2e_steps, e2e_step, max(args.warmup, 3)),
                                     dev)
        # the host results of the last replay are the kernels' results
        y_dev = K.spmv_csr(nrows, ncols, pos, crd, vals, x0)
        for s in range(min(ns, e2e_steps)):
            for r in bound[s].results:
                assert torch.equal(r.vals, y_dev.cpu()), "e2e host result differs from the kernel's"
        h2d_step, d2h_step = bound[0].h2d_bytes, bound[0].d2h_bytes
        e2e_val = D.sum_over_ranks(float(b_csr + b_ell), dev) / t_e2e / 1e9

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
            "config": headline_config(world, nrows, nnz, S),
            "timing": {"l2": timer.describe(), "operand_copies": {"csr": nc_csr, "ell": nc_ell},
                       "launch": dict(timer.method),
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
                    "h2d_bytes_per_step": int(h2d_step),
                    "d2h_bytes_per_step": int(d2h_step),
                    "ms_per_step": round(t_e2e * 1e3, 4),
                    "path": "compile_many([y = A_csr * x, y = A_ell * x]) bound once (public API), "
                            "one CUDA-graph launch per step: pinned host x -> device, both SpMV "
                            "kernels, both y packed and sent to pinned host in one copy, every "
                            "step; matrices resident in "
                            f"HBM; steps rotate over {ns} streams",
                    "timing": f"wall clock, synchronised both sides; median of 5 batches of "
                              f"{e2e_steps} steps after {max(args.warmup, 2 * ns)} warm-up steps",
                    "eager": {"value": round(D.sum_over_ranks(float(b_csr + b_ell), dev)
                                             / t_eager / 1e9, 3),
                              "ms_per_step": round(t_eager * 1e3, 4),
                              "path": "two evaluate() calls per step with the same copies "
                                      "(planning cached, launches from Python)"}},
            "gpu_launches": launches,
            "gpu_launches_note": (f"{launches} SpMV kernel launches inside the timed events "
                                  "(K CSR + K ELL)"),
        }

        # ---- optional all-gather of the y row blocks (N > 1), timed on its own:
        # the one data-path collective the north star allows after compute
        if world > 1:
            y1 = csr_ops[0][4]
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
        # blocks of the one D5 tensor (strong scaling: total work fixed).  Rank 0
        # generates the tensor and sends each rank its slice block over NCCL
        # (no rank but 0 materialises it); factors replicated by broadcast.
        if world > 1 and not args.no_formats:
            out["mttkrp_coo3_sharded"] = mttkrp_sharded(torch, dist, D, K, wl, dev, rank, world,
                                                        timer, clk)

        # ---- CPU baseline (rank 0, N = 1): the oracle port on the host cores
        if rank == 0 and world == 1:
            out["cpu_baseline"] = cpu_baseline(st, ell)

        # ---- the other BASELINE configs, same run (N = 1)
        if world == 1 and not args.no_formats:
            out["formats"] = run_formats(torch, K, F, wl, evaluate, compile_, dev, timer, peak, l2, clk,
                                         max(5, min(args.steps, 30)))
    out["clocks"] = clk.summary()
    out["clocks"]["headline_samples"] = clk.summary("headline")["samples"]
    out["clocks"]["note"] = ("NVML polled every 0.5 ms; samples from every timed region "
                             "(headline kernels, formats kernels, e2e loops)")
    return out


def mttkrp_sharded(torch, dist, D, K, wl, dev, rank, world, timer, clk):
    sizes = torch.zeros(world + 1, dtype=torch.int64, device=dev)
    dims = torch.zeros(4, dtype=torch.int64, device=dev)
    if rank == 0:
        mt = wl.mttkrp()
        I, J, Kd, R = mt["I"], mt["J"], mt["K"], mt["R"]
        sb = D.slice_blocks_coo3(mt["i"], I, world)
        ebounds = np.searchsorted(mt["i"], sb).astype(np.int64)
        sizes.copy_(torch.as_tensor(ebounds))
        dims.copy_(torch.as_tensor([I, J, Kd, R]))
        full = [torch.as_tensor(mt[k], device=dev) for k in ("i", "j", "k", "vals")]
        Bt = torch.as_tensor(mt["B"], device=dev).reshape(J, R)
        Ct = torch.as_tensor(mt["C"], device=dev).reshape(Kd, R)
        slices = torch.as_tensor(sb.astype(np.int64), device=dev)
        del mt
    else:
        slices = torch.zeros(world + 1, dtype=torch.int64, device=dev)
    dist.broadcast(sizes, 0)
    dist.broadcast(dims, 0)
    dist.broadcast(slices, 0)
    I, J, Kd, R = (int(v) for v in dims.tolist())
    e = [int(v) for v in sizes.tolist()]
    s0, s1 = int(slices[rank]), int(slices[rank + 1])
    n_loc = e[rank + 1] - e[rank]
    # NCCL sends device buffers directly; gloo (the multi-rank smoke test on a
    # 1-GPU box) only moves host tensors
    via_host = dist.get_backend() != "nccl"
    if rank == 0:
        loc = [t[e[0]:e[1]] for t in full]
        for r in range(1, world):
            for t in full:
                part = t[e[r]:e[r + 1]].contiguous()
                dist.send(part.cpu() if via_host else part, r)
    else:
        loc = [torch.empty(n_loc, dtype=torch.int32, device=dev) for _ in range(3)] + \
              [torch.empty(n_loc, dtype=torch.float64, device=dev)]
        for t in loc:
            if via_host:
                h = torch.empty(t.shape, dtype=t.dtype)
                dist.recv(h, 0)
                t.copy_(h)
            else:
                dist.recv(t, 0)
        Bt = torch.empty((J, R), dtype=torch.float64, device=dev)
        Ct = torch.empty((Kd, R), dtype=torch.float64, device=dev)
    D.replicate(Bt, src=0)
    D.replicate(Ct, src=0)
    ti, tj, tk, tv = loc
    ti = ti - s0                      # this rank's A rows are [s0, s1)
    At = torch.empty((s1 - s0, R), dtype=torch.float64, device=dev)
    ws = torch.empty(int(K.L().sl_mttkrp_workspace_bytes(n_loc, R)), dtype=torch.uint8,
                     device=dev)
    if rank == 0:
        del full
    dist.barrier()
    with clk.timed("mttkrp_sharded"):
        tm = timer.run({"mttkrp": [lambda: K.mttkrp_coo3(s1 - s0, J, Kd, ti, tj, tk, tv, Bt, Ct,
                                                         At, ws=ws)] * 2}, 10, 3)
    t_mt = D.max_over_ranks(float(tm["mttkrp"]), dev)      # ms
    nnz_all = D.sum_over_ranks(float(n_loc), dev)
    return {"ms": round(t_mt, 5), "nnz/s": round(nnz_all / (t_mt * 1e-3), 1),
            "nnz*R/s": round(nnz_all * R / (t_mt * 1e-3), 1),
            "GFLOP/s": round(3 * nnz_all * R / (t_mt * 1e-3) / 1e9, 1),
            "nnz_per_rank_max_over_mean": round(D.max_over_ranks(float(n_loc), dev)
                                                / (nnz_all / world), 4),
            "scaling": "strong",
            "note": "slice blocks balanced by nnz, sent from rank 0 over NCCL; B, C broadcast; "
                    "max over ranks of the mean launch time (the 811 MB tensor exceeds L2)"}


def cpu_baseline(st, ell):
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # test infrastructure: CPU baseline leg only

    thr = host_threads()
    nrows = st["nrows"]
    b = bytes_csr(nrows, len(st["crd"])) + bytes_ell(nrows, ell["nslots"])

    def step():
        oracle.spmv_csr(nrows, st["pos"], st["crd"], st["vals"], st["x"], threads=thr)
        oracle.spmv_ell(nrows, ell["nslots"], ell["crd"], ell["vals"], st["x"], threads=thr)

    dt, n = time_cpu(step, min_s=3.0)
    return {"value": round(b / dt / 1e9, 3), "unit": "GB/s", "cores": thr, "kind": "port",
            "sample": f"{n} steps of CSR+ELL SpMV on the full 64^3 stencil ({dt * 1e3:.2f} ms/step, "
                      f"{n * dt:.1f} s), C restatement of the reference (oracle/)",
            "cpu_model": cpu_model(), "host_cpu_count": os.cpu_count()}


def cpu_leg(label, fn, nbytes=None, units=None, unit_name=None, min_s=1.5):
    """Oracle (C port of the reference) timed on the host cores for a config."""
    dt, n = time_cpu(fn, min_s=min_s)
    d = {"ms": round(dt * 1e3, 3), "cores": host_threads(), "kind": "port",
         "sample": f"{n} full-size runs of {label} ({n * dt:.1f} s), oracle/ C restatement",
         "cpu_model": cpu_model()}
    if nbytes is not None:
        d["GB/s"] = round(nbytes / dt / 1e9, 3)
    if units is not None:
        d[unit_name] = round(units / dt, 1)
    return d


def run_formats(torch, K, F, wl, evaluate, compile_, dev, timer, peak, l2, clk, steps):
    """The other BASELINE configs: kernel time (rotating copies, one event pair
    per K launches), e2e through `evaluate` with host buffers, CPU baseline."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # test infrastructure: the CPU-baseline legs and the MTTKRP check only

    thr = host_threads()
    res = {}
    T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    ns = E2E_STREAMS
    streams = [torch.cuda.Stream(device=dev) for _ in range(ns)]

    def spmv_e2e(A_st, xh, nrows, nbytes):
        """One `compile`d step per pipeline slot (x copy node, the kernels of
        `evaluate`, y copy node in one graph); the eager two-call form beside it."""
        xs = [F.dense_storage(torch.as_tensor(xh).pin_memory(), device=None) for _ in range(ns)]
        ys = [torch.empty(nrows, dtype=torch.float64).pin_memory() for _ in range(ns)]
        expr = "y(i) = A(i,j) * x(j)"

        def eager(k):
            with torch.cuda.stream(streams[k % ns]):
                y = evaluate(expr, {"A": A_st, "x": xs[k % ns]}).vals
                ys[k % ns].copy_(y, non_blocking=True)
        bound = [compile_(expr, {"A": A_st, "x": xs[s]}) for s in range(ns)]

        def step(k):
            bound[k % ns](streams[k % ns])
        with clk.timed("e2e"):
            te = e2e_loop(torch, 50, eager)
            t = e2e_loop(torch, 50, step)
        assert torch.equal(bound[0].results[0].vals, ys[0]), "compiled e2e result != eager"
        return {"GB/s": round(nbytes / t / 1e9, 3), "ms_per_step": round(t * 1e3, 4),
                "h2d_bytes_per_step": bound[0].h2d_bytes, "d2h_bytes_per_step": bound[0].d2h_bytes,
                "path": "compile(evaluate) bound once, one graph launch per step: pinned host x "
                        "in, y out; matrix resident in HBM",
                "eager": {"GB/s": round(nbytes / te / 1e9, 3), "ms_per_step": round(te * 1e3, 4),
                          "path": "evaluate() per step with the same copies"}}

    # ---- D1: COO SpMV on unconverted coordinates (+ the paper's convert-then-CSR)
    d = wl.coo_spmv()
    n, m, nnz = d["nrows"], d["ncols"], len(d["rows"])
    b = bytes_coo(n, m, nnz)
    ycpu = np.empty(n)
    ops = dev_copies(torch, (d["rows"], d["cols"], d["vals"], d["x"], ycpu), copies_for(b, l2), dev)
    pos_h = wl.coo_to_csr_pos(d["rows"], n)
    csr_ops = dev_copies(torch, (pos_h, d["cols"], d["vals"], d["x"], ycpu),
                         copies_for(bytes_csr(n, nnz), l2), dev)
    rp = [torch.empty(n + 1, dtype=torch.int32, device=dev) for _ in range(len(ops))]
    with clk.timed("formats"):
        tt = timer.run({"coo": [lambda o=o: K.spmv_coo(n, m, *o) for o in ops],
                        "csr": [lambda o=o: K.spmv_csr(n, m, *o) for o in csr_ops],
                        "conv": [lambda o=o: K.coo_to_csr(n, o[0], o[1], o[2], sync=False)
                                 for o in ops],
                        "rowptr": [lambda o=o, r=r: K.coo_rowptr(n, o[0], r)
                                   for o, r in zip(ops, rp)]}, steps, 3)
    t = tt["coo"]
    g8 = l2_calib().get("gather8_20M_G_per_s") or l2_calib().get("gather8_G_per_s")
    res["coo_spmv_D1"] = {
        "ms": round(t, 5), "GB/s": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / peak, 4),
        "nnz/s": round(nnz / t * 1e3, 1), "bytes": b, "copies": len(ops),
        "gather_ceiling": {"x_gathers": nnz, "peak_G_per_s": g8,
                           "floor_ms": round(nnz / g8 / 1e6, 5) if g8 else None},
        "e2e": spmv_e2e(F.coo_storage(ops[0][0], ops[0][1], ops[0][2], (n, m), device=dev),
                        d["x"], n, b),
        "cpu_baseline": cpu_leg("COO SpMV D1", lambda: oracle.spmv_coo(
            n, d["rows"], d["cols"], d["vals"], d["x"], threads=thr), nbytes=b)}
    bs = bytes_csr(n, nnz)
    res["csr_spmv_D1"] = {"ms": round(tt["csr"], 5), "GB/s": round(bs / tt["csr"] / 1e6, 1),
                          "frac": round(bs / tt["csr"] / 1e6 / peak, 4), "bytes": bs}
    bc = 16 * nnz + 4 * (n + 1) + 12 * nnz
    res["convert_coo_to_csr_D1"] = {"ms": round(tt["conv"], 5),
                                    "GB/s": round(bc / tt["conv"] / 1e6, 1),
                                    "frac": round(bc / tt["conv"] / 1e6 / peak, 4), "bytes": bc}
    br = 4 * nnz + 4 * (n + 1)
    res["coo_rowptr_D1"] = {"ms": round(tt["rowptr"], 5), "GB/s": round(br / tt["rowptr"] / 1e6, 1),
                            "bytes": br}
    # the paper's end-to-end question (Fig. 13): COO SpMV on unconverted
    # coordinates vs converting to CSR first (exact identity copy) and then CSR SpMV
    res["coo_vs_convert_then_csr_D1"] = {
        "coo_spmv_ms": res["coo_spmv_D1"]["ms"],
        "convert_plus_csr_ms": round(tt["conv"] + tt["csr"], 5),
        "rowptr_only_plus_csr_ms": round(tt["rowptr"] + tt["csr"], 5)}

    # ---- H1: CSR x hashed x (per-nonzero probing, and the slot map)
    h = wl.hash_vector()
    hc, hv = T(h["crd"]), T(h["vals"])
    hws = torch.empty(int(K.L().sl_spmv_csr_hashx_map_workspace_bytes(m, h["width"])),
                      dtype=torch.uint8, device=dev)
    with clk.timed("formats"):
        tt = timer.run({"probe": [lambda o=o: K.spmv_csr_hashx(n, o[0], o[1], o[2], h["width"],
                                                               hc, hv, o[4])
                                  for o in csr_ops[:2]],
                        "map": [lambda o=o: K.spmv_csr_hashx(n, o[0], o[1], o[2], h["width"], hc,
                                                             hv, o[4], n=m, ws=hws)
                                for o in csr_ops]}, steps, 3)
    bh = 4 * (n + 1) + 12 * nnz + 8 * n + 12 * h["width"]
    res["csr_hashx_H1"] = {"ms": round(tt["probe"], 5), "GB/s": round(bh / tt["probe"] / 1e6, 1),
                           "frac": round(bh / tt["probe"] / 1e6 / peak, 4),
                           "locates/s": round(nnz / tt["probe"] * 1e3, 1), "bytes": bh,
                           "path": "per-nonzero warp-cooperative probing",
                           "note": "H1's table (c mod 131072 over coordinates in [0, 200000)) "
                                   "holds one 20.6K-slot probe cluster: mean probe length 1963 "
                                   "over all coordinates (max 20.5K), so this path reads ~3.9G "
                                   "slots per SpMV; evaluate() resolves each coordinate once "
                                   "(slot map, next entry) whenever nnz >= table width"}
    res["csr_hashx_map_H1"] = {"ms": round(tt["map"], 5), "GB/s": round(bh / tt["map"] / 1e6, 1),
                               "frac": round(bh / tt["map"] / 1e6 / peak, 4),
                               "locates/s": round(nnz / tt["map"] * 1e3, 1), "bytes": bh,
                               "path": "slot map (one locate per coordinate) + CSR SpMV",
                               "cpu_baseline": cpu_leg("CSR x hash-x H1", lambda: oracle.spmv_csr_hashx(
                                   n, pos_h, d["cols"], d["vals"], h["width"], h["crd"], h["vals"],
                                   threads=thr), units=nnz, unit_name="locates/s")}
    del ops, csr_ops, rp, hws

    # ---- widened patterns on the headline stencil
    st = wl.stencil27()
    n, nnz = st["nrows"], len(st["crd"])
    Kc = 16
    rng = np.random.default_rng(5)
    Xd = rng.uniform(-1, 1, (n, Kc))
    keep = np.sort(rng.choice(n, n // 2, replace=False)).astype(np.int32)
    xkv = rng.uniform(-1, 1, len(keep))
    b_spmm = 4 * (n + 1) + 12 * nnz + 16 * n * Kc
    mops = dev_copies(torch, (st["pos"], st["crd"], st["vals"], Xd, np.empty((n, Kc))),
                      copies_for(b_spmm, l2), dev)
    b_spx = 4 * (n + 1) + 12 * nnz + 12 * len(keep) + 8 * n
    xops = dev_copies(torch, (st["pos"], st["crd"], st["vals"], keep, xkv, np.empty(n)),
                      copies_for(b_spx, l2), dev)
    sws = torch.empty(int(K.L().sl_spmv_csr_spx_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    with clk.timed("formats"):
        tt = timer.run({"spmm": [lambda o=o: K.spmm_csr(n, n, *o) for o in mops],
                        "spx": [lambda o=o: K.spmv_csr_spx(n, n, *o, sws) for o in xops]},
                       steps, 3)
    t = tt["spmm"]
    res["spmm_csr_stencil_K16"] = {"ms": round(t, 5), "GB/s": round(b_spmm / t / 1e6, 1),
                                   "frac": round(b_spmm / t / 1e6 / peak, 4), "bytes": b_spmm,
                                   "GFLOP/s": round(2 * nnz * Kc / t / 1e6, 1)}
    t = tt["spx"]
    res["spmv_csr_spx_stencil"] = {"ms": round(t, 5), "GB/s": round(b_spx / t / 1e6, 1),
                                   "frac": round(b_spx / t / 1e6 / peak, 4), "bytes": b_spx,
                                   "x_nnz": int(len(keep))}
    del mops, xops, sws
    # the paper's SpDM on COO (row pointer per call + SpMM), D1's matrix, K = 16
    dd = wl.coo_spmv()
    nd, md, nnzd = dd["nrows"], dd["ncols"], len(dd["rows"])
    Xc = rng.uniform(-1, 1, (md, Kc))
    b_sd = 16 * nnzd + 8 * md * Kc + 8 * nd * Kc
    sdops = dev_copies(torch, (dd["rows"], dd["cols"], dd["vals"], Xc, np.empty((nd, Kc))),
                       copies_for(b_sd, l2), dev)

    def spdm(o):
        pos = K.coo_rowptr(nd, o[0])
        K.spmm_csr(nd, md, pos, o[1], o[2], o[3], o[4])

    with clk.timed("formats"):
        tt = timer.run({"spdm": [lambda o=o: spdm(o) for o in sdops]}, steps, 3)
    t = tt["spdm"]
    res["spdm_coo_D1_K16"] = {"ms": round(t, 5), "GB/s": round(b_sd / t / 1e6, 1),
                              "frac": round(b_sd / t / 1e6 / peak, 4), "bytes": b_sd,
                              "GFLOP/s": round(2 * nnzd * Kc / t / 1e6, 1)}
    del sdops

    # ---- D3: DIA SpMV
    g = wl.dia7()
    n = g["nrows"]
    b = bytes_dia(n, n, g["offsets"].tolist())
    offs = g["offsets"]
    ops = dev_copies(torch, (g["vals"], g["x"], np.empty(n)), copies_for(b, l2), dev)
    with clk.timed("formats"):
        tt = timer.run({"dia": [lambda o=o: K.spmv_dia(n, n, offs, *o) for o in ops]}, steps, 3)
    t = tt["dia"]
    res["dia_spmv_D3"] = {
        "ms": round(t, 5), "GB/s": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / peak, 4),
        "bytes": b, "copies": len(ops),
        "e2e": spmv_e2e(F.dia_storage(offs, ops[0][0], (n, n), device=dev), g["x"], n, b),
        "cpu_baseline": cpu_leg("DIA SpMV D3", lambda: oracle.spmv_dia(
            n, n, offs, g["vals"], g["x"], threads=thr), nbytes=b)}
    del ops

    # ---- D4: C = A + B (CSR + COO -> CSR)
    a = wl.add_ab()
    n = a["nrows"]
    ops = dev_copies(torch, (a["a_pos"], a["a_crd"], a["a_vals"], a["b_rows"], a["b_cols"],
                             a["b_vals"]), 2, dev)
    outs = {}

    def add(o):
        outs["c"] = K.add_csr(n, o[0], o[1], o[2], o[4], o[5], b_rows=o[3], sync=False)

    with clk.timed("formats"):
        tt = timer.run({"add": [lambda o=o: add(o) for o in ops]}, steps, 3)
    nnz_c = int(outs["c"][0][n].item())
    b = 4 * (n + 1) + 12 * len(a["a_crd"]) + 16 * len(a["b_cols"]) + 4 * (n + 1) + 12 * nnz_c
    t = tt["add"]
    nin = len(a["a_crd"]) + len(a["b_cols"])
    # e2e: both operands from pinned host memory, C (pos, crd, vals) back
    A_h = F.csr_storage(torch.as_tensor(a["a_pos"]), torch.as_tensor(a["a_crd"]),
                        torch.as_tensor(a["a_vals"]).pin_memory(), (n, n), device=None)
    B_h = F.coo_storage(torch.as_tensor(a["b_rows"]), torch.as_tensor(a["b_cols"]),
                        torch.as_tensor(a["b_vals"]).pin_memory(), (n, n), device=None)
    for lv in A_h.levels + B_h.levels:
        for attr in ("pos", "crd"):
            v = getattr(lv, attr)
            if v is not None:
                setattr(lv, attr, v.pin_memory())
    c_host = {}

    def add_step(k):
        C = evaluate("C(i,j) = A(i,j) + B(i,j)", {"A": A_h.to(dev, non_blocking=True),
                                                 "B": B_h.to(dev, non_blocking=True)},
                     F.preset("csr"))
        c_host["pos"] = C.levels[1].pos.to("cpu", non_blocking=True)
        c_host["crd"] = C.levels[1].crd.to("cpu", non_blocking=True)
        c_host["vals"] = C.vals.to("cpu", non_blocking=True)

    with clk.timed("e2e"):
        t_e2e = e2e_loop(torch, 5, add_step, warmup=2, batches=3)
    h2d = sum(int(v.numel() * v.element_size()) for st_ in (A_h, B_h)
              for v in [st_.vals] + [getattr(lv, a_) for lv in st_.levels
                                     for a_ in ("pos", "crd") if getattr(lv, a_) is not None])
    d2h = 4 * (n + 1) + 12 * nnz_c
    res["add_csr_coo_D4"] = {
        "ms": round(t, 5), "GB/s": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / peak, 4),
        "nnz_c": nnz_c, "bytes": b, "input nnz/s": round(nin / t * 1e3, 1), "copies": 2,
        "e2e": {"GB/s": round(b / t_e2e / 1e9, 3), "input nnz/s": round(nin / t_e2e, 1),
                "ms_per_step": round(t_e2e * 1e3, 3), "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "evaluate('C(i,j) = A(i,j) + B(i,j)', csr) with A (CSR) and B (COO) "
                        "copied from pinned host memory and C read back every step"},
        "cpu_baseline": cpu_leg("A+B D4", lambda: oracle.add_csr(
            n, a["a_pos"], a["a_crd"], a["a_vals"], a["b_cols"], a["b_vals"], b_rows=a["b_rows"],
            threads=thr), nbytes=b, units=nin, unit_name="input nnz/s")}
    del ops, outs, A_h, B_h, c_host

    # ---- D5: MTTKRP over COO-3 and CSF (+ TTV / INNERPROD on the same tensor)
    mt = wl.mttkrp()
    csf = wl.coo3_to_csf(mt["i"], mt["j"], mt["k"], None)
    I, J, Kd, R = mt["I"], mt["J"], mt["K"], mt["R"]
    nnz = len(mt["i"])
    ti, tj, tk, tv = T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"])
    Bt, Ct = T(mt["B"]).reshape(J, R), T(mt["C"]).reshape(Kd, R)
    c0, p1, c1, p2, c2 = (T(csf[k]) for k in ("crd0", "pos1", "crd1", "pos2", "crd2"))
    A = torch.empty((I, R), dtype=torch.float64, device=dev)
    ws = torch.empty(int(K.L().sl_mttkrp_workspace_bytes(nnz, R)), dtype=torch.uint8, device=dev)
    # the tensor (811 / 533 MB) exceeds L2 several times: two launches
    # alternate over two copies of the factors (B, C, A), the tensor is shared
    Bt2, Ct2, A2 = Bt.clone(), Ct.clone(), torch.empty_like(A)
    fc = [(Bt, Ct, A), (Bt2, Ct2, A2)]
    with clk.timed("formats"):
        tt = timer.run({"coo3": [lambda f=f: K.mttkrp_coo3(I, J, Kd, ti, tj, tk, tv, *f, ws)
                                 for f in fc],
                        "csf": [lambda f=f: K.mttkrp_csf(I, J, Kd, c0, p1, c1, p2, c2, tv, *f, ws)
                                for f in fc]},
                       max(3, steps // 3), 2)
    bf = 8 * (J * R + Kd * R + I * R)
    b_coo = 20 * nnz + bf
    n1 = len(csf["crd1"])
    b_csf = 8 + 4 * len(csf["crd0"]) + 4 * (len(csf["crd0"]) + 1) + 4 * n1 + 4 * (n1 + 1) + 12 * nnz + bf
    l2c = l2_calib()
    l2_peak = l2c.get("gather256_GBs")
    l2_rows = 8 * R * (nnz + n1) + 8 * I * R
    # the check (oracle as the checker): the reference's sequential order,
    # strict |d| <= 1e-12 |ref| and the condition-scaled bound per component
    A_gpu = K.mttkrp_coo3(I, J, Kd, ti, tj, tk, tv, Bt, Ct).cpu().numpy()
    A_ref, A_abs = oracle.mttkrp_coo3(I, mt["i"], mt["j"], mt["k"], mt["vals"],
                                      mt["B"].reshape(J, R), mt["C"].reshape(Kd, R))
    dlt = np.abs(A_gpu - A_ref)
    check = {"components": int(A_ref.size),
             "strict_rtol_1e-12_pass": int(np.sum(dlt <= 1e-12 * np.abs(A_ref))),
             "condition_scaled_1e-12_pass": int(np.sum(dlt <= 1e-12 * np.maximum(np.abs(A_ref),
                                                                                 A_abs))),
             "bit_identical": int(np.sum(A_gpu.view(np.int64) == A_ref.view(np.int64)))}
    cpu_mt = cpu_leg("MTTKRP COO-3 D5", lambda: oracle.mttkrp_coo3(
        I, mt["i"], mt["j"], mt["k"], mt["vals"], mt["B"].reshape(J, R), mt["C"].reshape(Kd, R),
        threads=thr), nbytes=b_coo, units=nnz, unit_name="nnz/s", min_s=2.0)
    # e2e: X resident (the tensor of a CP-ALS run), the factors in from pinned
    # host memory and A out every step
    X_st = F.coo3_storage(ti, tj, tk, tv, (I, J, Kd), device=dev)
    Bh = [torch.as_tensor(mt["B"]).pin_memory() for _ in range(ns)]
    Ch = [torch.as_tensor(mt["C"]).pin_memory() for _ in range(ns)]
    Ah = [torch.empty(I * R, dtype=torch.float64).pin_memory() for _ in range(ns)]

    def mt_step(k):
        with torch.cuda.stream(streams[k % ns]):
            Bs = F.dense_storage(Bh[k % ns].to(dev, non_blocking=True), (J, R), device=None)
            Cs = F.dense_storage(Ch[k % ns].to(dev, non_blocking=True), (Kd, R), device=None)
            Ao = evaluate("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)", {"X": X_st, "B": Bs, "C": Cs})
            Ah[k % ns].copy_(Ao.vals, non_blocking=True)

    mt_bound = [compile_("A(i,r) = X(i,j,k) * B(j,r) * C(k,r)",
                         {"X": X_st, "B": F.dense_storage(Bh[s], (J, R), device=None),
                          "C": F.dense_storage(Ch[s], (Kd, R), device=None)}) for s in range(ns)]

    def mt_bound_step(k):
        mt_bound[k % ns](streams[k % ns])

    with clk.timed("e2e"):
        t_eager = e2e_loop(torch, 10, mt_step, warmup=2, batches=3)
        t_e2e = e2e_loop(torch, 10, mt_bound_step, warmup=2, batches=3)
    assert torch.equal(mt_bound[0].results[0].vals, Ah[0].reshape(-1)), "compiled MTTKRP != eager"
    for name, b, key in (("mttkrp_coo3_D5", b_coo, "coo3"), ("mttkrp_csf_D5", b_csf, "csf")):
        t = tt[key]
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
    res["mttkrp_coo3_D5"]["check_vs_oracle"] = check
    res["mttkrp_coo3_D5"]["cpu_baseline"] = cpu_mt
    res["mttkrp_coo3_D5"]["e2e"] = {
        "nnz/s": round(nnz / t_e2e, 1), "ms_per_step": round(t_e2e * 1e3, 3),
        "h2d_bytes_per_step": 8 * (J + Kd) * R, "d2h_bytes_per_step": 8 * I * R,
        "path": "compile('A(i,r) = X(i,j,k) * B(j,r) * C(k,r)') bound once, one graph launch per "
                "step: X COO-3 resident, B and C in from pinned host memory, A out, every step",
        "eager": {"nnz/s": round(nnz / t_eager, 1), "ms_per_step": round(t_eager * 1e3, 3)}}
    del A_gpu, A_ref, A_abs, Bt2, Ct2, A2

    # the paper's other kernels on the same tensor: TTV into a
    # CSR-over-fibers output and INNERPROD of the COO-3 tensor with itself
    vt = T(np.random.default_rng(3).uniform(-1.0, 1.0, Kd))
    zi, zj, zk, zv = ti.clone(), tj.clone(), tk.clone(), tv.clone()
    with clk.timed("formats"):
        tt = timer.run({"ttv": [lambda: K.ttv_csf(I, J, Kd, c0, p1, c1, p2, c2, tv, vt,
                                                  out="csr")] * 2,
                        "inner": [lambda: K.inner_coo3(I, J, Kd, (ti, tj, tk, tv),
                                                       (zi, zj, zk, zv))] * 2},
                       max(3, steps // 3), 2)
    t = tt["ttv"]
    b_ttv = (4 * (len(csf["crd0"]) + 1) + 4 * len(csf["crd0"]) + 4 * (n1 + 1) + 12 * nnz + 8 * Kd
             + 4 * (I + 1) + 12 * n1)
    res["ttv_csf_csr_out_D5"] = {"ms": round(t, 4), "GB/s": round(b_ttv / t / 1e6, 1),
                                 "frac": round(b_ttv / t / 1e6 / peak, 4), "bytes": b_ttv,
                                 "nnz/s": round(nnz / t * 1e3, 1), "fibers": n1}
    t = tt["inner"]
    b_in = 2 * 20 * nnz
    res["innerprod_coo3_D5"] = {"ms": round(t, 4), "GB/s": round(b_in / t / 1e6, 1),
                                "frac": round(b_in / t / 1e6 / peak, 4), "bytes": b_in,
                                "nnz/s": round(nnz / t * 1e3, 1)}

    # 3rd-order PLUS through `evaluate`: X = D5 (COO-3) plus Z =
    # every other nonzero of it with new values, into COO-3
    X_st = F.coo3_storage(ti, tj, tk, tv, (I, J, Kd), device=dev)
    Z_st = F.coo3_storage(ti[::2].contiguous(), tj[::2].contiguous(), tk[::2].contiguous(),
                          (tv[::2] * 0.5).contiguous(), (I, J, Kd), device=dev)
    out = {}

    def plus3():
        out["c"] = evaluate("A(i,j,k) = X(i,j,k) + Z(i,j,k)", {"X": X_st, "Z": Z_st},
                            F.preset("coo-3"))

    with clk.timed("formats"):
        tt = timer.run({"plus3": [plus3, plus3]}, 3, 2, capture=False)
    nz_c = int(out["c"].levels[2].crd.numel())
    b_p = 20 * nnz + 20 * (nnz // 2) + 20 * nz_c
    res["plus3_coo3_D5"] = {"ms": round(tt["plus3"], 4), "GB/s": round(b_p / tt["plus3"] / 1e6, 1),
                            "frac": round(b_p / tt["plus3"] / 1e6 / peak, 4), "bytes": b_p,
                            "nnz_c": nz_c, "launch": timer.method.get("plus3"),
                            "path": "evaluate(): union of the operands' fibres, long fibres cut into "
                                    "k-blocks, the A + B kernels over (fibre block x k); torch "
                                    "glue for the keys, host syncs for the output sizes"}
    del X_st, Z_st, out
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
    thr = host_threads()
    nrows, nnz = st["nrows"], len(st["crd"])
    b = bytes_csr(nrows, nnz) + bytes_ell(nrows, ell["nslots"])

    def one():
        oracle.spmv_csr(nrows, st["pos"], st["crd"], st["vals"], st["x"], threads=thr)
        oracle.spmv_ell(nrows, ell["nslots"], ell["crd"], ell["vals"], st["x"], threads=thr)

    # a step is a bounded sample of the workload: `reps` CSR+ELL SpMVs, sized
    # so one step takes ~100 ms (the whole K-step run stays well above a
    # second for any K the driver uses, and within a few minutes for K <= 1000)
    t0 = time.perf_counter()
    for _ in range(3):
        one()
    t1 = (time.perf_counter() - t0) / 3
    reps = max(1, int(0.1 / max(t1, 1e-6)))
    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(reps):
            one()
    dt = (time.perf_counter() - t0) / (args.steps * reps)
    value = b / dt / 1e9
    S = ell["nslots"]
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * reps * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy; BASELINE configs have no public dataset)",
        "config": headline_config(world, nrows // world, nnz // world, S),
        "timing": {"parallelism": f"host threads x{thr} (the whole grid on rank 0)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": thr, "kind": "port",
                         "sample": f"{args.steps} steps x {reps} CSR+ELL SpMVs of the full grid "
                                   f"({dt * reps * args.steps:.1f} s); C restatement of the "
                                   "reference (the Python reference is absent on the GPU box)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
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
