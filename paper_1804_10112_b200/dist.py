"""Multi-GPU partitioning of the hot path.

SpMV and MTTKRP shard by contiguous, nnz-balanced blocks of output rows
(slices): each rank owns rows [r0, r1), computes its block of y (A) with no
data-path exchange, and reads a replicated x (B, C).  torch.distributed
over NCCL is used only to replicate x / the factors once (broadcast) and,
optionally, to gather the row blocks of y back (all-gather of padded
blocks).  One process per GPU.

`evaluate_sharded` is the public multi-GPU entry: every rank passes the same
global operands (resident on its own device); the row blocks are cut on the
device (searchsorted on the row pointer / row coordinates), each rank's
shard is a view or a device-side slice of the operand, the rank evaluates its
block with the single-GPU `evaluate`, and the blocks are optionally
all-gathered.  The numpy partition/shard helpers below serve the bench and
the host-side tests; everything is covered by world_size-2 gloo tests on CPU
(tests/test_dist_gloo.py) — there the per-rank evaluation is injected (the C
oracle), on a GPU box it is the sm_100a kernels.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np


def balanced_row_blocks(row_nnz_prefix: np.ndarray, nparts: int) -> np.ndarray:
    """Boundaries b[0]=0 <= ... <= b[nparts]=nrows of contiguous row blocks
    with roughly equal nonzeros.  `row_nnz_prefix` is a CSR-style pos array
    (length nrows+1).  Block p ends at the first row whose prefix reaches
    p/nparts of the total (searchsorted on pos)."""
    pos = np.asarray(row_nnz_prefix, dtype=np.int64)
    nrows = len(pos) - 1
    total = int(pos[-1])
    b = np.zeros(nparts + 1, dtype=np.int64)
    for p in range(1, nparts):
        target = (total * p) // nparts
        b[p] = min(max(int(np.searchsorted(pos, target, side="left")), b[p - 1]), nrows)
    b[nparts] = nrows
    return b


def coo_row_blocks(rows: np.ndarray, nrows: int, nparts: int) -> np.ndarray:
    """Row blocks for a row-sorted COO: element cut points snapped to row starts."""
    counts = np.bincount(np.asarray(rows, dtype=np.int64), minlength=nrows)
    pos = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=pos[1:])
    return balanced_row_blocks(pos, nparts)


@dataclass
class RowShard:
    rank: int
    r0: int
    r1: int

    @property
    def nrows(self) -> int:
        return self.r1 - self.r0


def shard_csr(pos, crd, vals, r0, r1):
    pos = np.asarray(pos, dtype=np.int64)
    lo, hi = int(pos[r0]), int(pos[r1])
    return (pos[r0:r1 + 1] - lo).astype(np.int32), np.asarray(crd)[lo:hi], np.asarray(vals)[lo:hi]


def shard_coo(rows, cols, vals, r0, r1):
    rows = np.asarray(rows)
    lo = int(np.searchsorted(rows, r0, side="left"))
    hi = int(np.searchsorted(rows, r1, side="left"))
    return (rows[lo:hi] - r0).astype(np.int32), np.asarray(cols)[lo:hi], np.asarray(vals)[lo:hi]


def shard_ell(nslots, crd, vals, nrows, r0, r1):
    """Slot-major ELL rows [r0, r1): slot s keeps positions s*N + [r0, r1)."""
    c = np.asarray(crd).reshape(nslots, nrows)[:, r0:r1]
    v = np.asarray(vals).reshape(nslots, nrows)[:, r0:r1]
    return np.ascontiguousarray(c).reshape(-1), np.ascontiguousarray(v).reshape(-1)


def shard_dia(offsets, vals, nrows, r0, r1):
    """DIA rows [r0, r1): each stored diagonal keeps its [r0, r1) slots; the
    offsets are unchanged and the kernel is told the global first row."""
    v = np.asarray(vals).reshape(len(offsets), nrows)[:, r0:r1]
    return np.asarray(offsets, dtype=np.int32), np.ascontiguousarray(v).reshape(-1)


def slice_blocks_coo3(i: np.ndarray, I: int, nparts: int) -> np.ndarray:
    """Slice (mode-0 row) blocks of a sorted COO-3 tensor, nnz-balanced."""
    return coo_row_blocks(i, I, nparts)


def shard_coo3(i, j, k, vals, s0, s1):
    i = np.asarray(i)
    lo = int(np.searchsorted(i, s0, side="left"))
    hi = int(np.searchsorted(i, s1, side="left"))
    return ((i[lo:hi] - s0).astype(np.int32), np.asarray(j)[lo:hi], np.asarray(k)[lo:hi],
            np.asarray(vals)[lo:hi])


def gather_row_blocks(y_local, bounds: Sequence[int], group=None):
    """All-gather of disjoint row blocks of y (uneven sizes padded to the
    largest block); returns the full vector on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [int(bounds[p + 1] - bounds[p]) for p in range(world)]
    m = max(sizes)
    if all(sz == m for sz in sizes) and y_local.is_contiguous():
        # equal blocks (the weak-scaling slabs): one collective, no copies
        full = torch.empty(m * world, dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(full, y_local, group=group)
        return full
    pad = torch.zeros(m, dtype=y_local.dtype, device=y_local.device)
    pad[:y_local.numel()] = y_local
    flat = torch.empty(m * world, dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(flat, pad, group=group)
    if not any(sz < m for sz in sizes):
        return flat
    keep = torch.cat([torch.arange(p * m, p * m + sizes[p], device=y_local.device)
                      for p in range(world)])
    return flat.index_select(0, keep)


def shard_add(a_pos, a_crd, a_vals, b_rows, b_cols, b_vals, r0, r1):
    """Row block [r0, r1) of C = A + B's operands (A CSR, B row-sorted COO):
    each rank computes its block of C with no exchange."""
    a = shard_csr(a_pos, a_crd, a_vals, r0, r1)
    b = shard_coo(b_rows, b_cols, b_vals, r0, r1)
    return a, b


def concat_csr_blocks(pos_local, crd_local, vals_local, group=None):
    """Assemble the global CSR of row-blocked results on every rank: an
    all-gather of the per-rank nnz totals gives each block's offset (the
    exclusive scan SURVEY.md §8(e) names), then the blocks' arrays are
    all-gathered (padded to the largest block)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = crd_local.device
    nnz = torch.tensor([crd_local.numel(), pos_local.numel() - 1], dtype=torch.int64, device=dev)
    sizes = [torch.empty_like(nnz) for _ in range(world)]
    dist.all_gather(sizes, nnz, group=group)
    nnzs = [int(t[0]) for t in sizes]
    rows = [int(t[1]) for t in sizes]
    offs = np.concatenate([[0], np.cumsum(nnzs)])

    def gather_padded(t, counts):
        m = max(max(counts), 1)
        pad = torch.zeros(m, dtype=t.dtype, device=dev)
        pad[:t.numel()] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        return [parts[p][:counts[p]] for p in range(world)]

    crd = torch.cat(gather_padded(crd_local, nnzs))
    vals = torch.cat(gather_padded(vals_local, nnzs))
    pos_parts = gather_padded(pos_local[1:].to(torch.int64), rows)
    pos = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev)] +
                    [pos_parts[p] + int(offs[p]) for p in range(world)])
    return pos.to(torch.int32), crd, vals


def replicate(t, src: int = 0, group=None):
    """Broadcast x (or a factor matrix) from `src` to every rank."""
    import torch.distributed as dist

    dist.broadcast(t, src=src, group=group)
    return t


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def shards_for(bounds: np.ndarray) -> List[RowShard]:
    return [RowShard(p, int(bounds[p]), int(bounds[p + 1])) for p in range(len(bounds) - 1)]


# ---------------------------------------------------------------------------
# public multi-GPU evaluation: device-side row blocks through `evaluate`

def _world(group):
    import torch.distributed as dist

    if not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _cuts(prefix, nparts: int):
    """Indices b[p] = first index with prefix[b] >= total * p / nparts (device
    searchsorted), b[0] = 0, b[nparts] = len(prefix) - 1."""
    import torch

    total = int(prefix[-1]) if prefix.numel() else 0
    n = prefix.numel() - 1
    tgt = torch.tensor([(total * p) // nparts for p in range(1, nparts)], dtype=prefix.dtype,
                       device=prefix.device)
    mid = torch.searchsorted(prefix, tgt).clamp_(max=n).tolist() if nparts > 1 else []
    b = [0] + [int(v) for v in mid] + [n]
    for p in range(1, len(b)):
        b[p] = max(b[p], b[p - 1])
    return b


def _coo_row_prefix_cuts(rows, nrows: int, nparts: int):
    """Row blocks of a row-sorted coordinate list, balanced by nonzeros:
    element cut points snapped back to their row's first element."""
    import torch

    nnz = rows.numel()
    if nparts == 1:
        return [0, nrows]
    if nnz == 0:
        return [(nrows * p) // nparts for p in range(nparts + 1)]
    idx = torch.tensor([(nnz * p) // nparts for p in range(1, nparts)], dtype=torch.int64,
                       device=rows.device).clamp_(max=nnz - 1)
    r = rows.to(torch.int64)[idx].tolist()
    b = [0] + [int(v) for v in r] + [nrows]
    for p in range(1, len(b)):
        b[p] = min(max(b[p], b[p - 1]), nrows)
    return b


def row_blocks(st, fmt_class: str, nparts: int, mode_dim: int):
    """Boundaries r[0] = 0 <= ... <= r[nparts] = n of contiguous blocks of the
    operand's first mode, balanced by stored nonzeros (ELL / DIA / dense:
    equal rows)."""
    import torch

    n = mode_dim
    if fmt_class == "csr":
        return _cuts(st.levels[1].pos.to(torch.int64), nparts)
    if fmt_class in ("coo", "coo3"):
        return _coo_row_prefix_cuts(st.levels[0].crd, n, nparts)
    if fmt_class == "csf":
        lv0, lv1, lv2 = st.levels
        leaf = lv2.pos.to(torch.int64)[lv1.pos.to(torch.int64)]     # nnz before each slice
        sb = _cuts(leaf, nparts)                                    # slice cut points
        crd0 = lv0.crd.to(torch.int64)
        return [0] + [int(crd0[s]) if s < crd0.numel() else n for s in sb[1:-1]] + [n]
    return [(n * p) // nparts for p in range(nparts + 1)]


def shard_storage(st, fmt_class: str, r0: int, r1: int):
    """Rows [r0, r1) of the operand's first mode as a storage of r1 - r0 rows
    (coordinates shifted by -r0), on the operand's device: views of the
    contiguous ranges for CSR / COO / COO-3 / CSF, a strided copy for ELL and
    DIA (their positions are slot- / diagonal-major)."""
    import torch

    from .formats import TensorStorage
    from .levels import LevelStorage

    dims = (r1 - r0,) + tuple(st.dims[1:])
    dev = st.vals.device
    L = st.levels
    if fmt_class == "csr":
        pos = L[1].pos
        lo, hi = int(pos[r0]), int(pos[r1])
        l0 = LevelStorage(L[0].spec, n=r1 - r0, device=dev)
        l1 = LevelStorage(L[1].spec, pos=(pos[r0:r1 + 1] - lo), crd=L[1].crd[lo:hi], device=dev)
        return TensorStorage(st.format, dims, [l0, l1], st.vals[lo:hi])
    if fmt_class in ("coo", "coo3"):
        rows = L[0].crd
        lo = int(torch.searchsorted(rows, torch.tensor([r0], dtype=rows.dtype, device=dev)))
        hi = int(torch.searchsorted(rows, torch.tensor([r1], dtype=rows.dtype, device=dev)))
        l0 = LevelStorage(L[0].spec, pos=[0, hi - lo], crd=rows[lo:hi] - r0, device=dev)
        rest = [LevelStorage(lv.spec, crd=lv.crd[lo:hi], device=dev) for lv in L[1:]]
        return TensorStorage(st.format, dims, [l0] + rest, st.vals[lo:hi])
    if fmt_class == "csf":
        crd0 = L[0].crd
        s0 = int(torch.searchsorted(crd0, torch.tensor([r0], dtype=crd0.dtype, device=dev)))
        s1 = int(torch.searchsorted(crd0, torch.tensor([r1], dtype=crd0.dtype, device=dev)))
        f0, f1 = int(L[1].pos[s0]), int(L[1].pos[s1])
        e0, e1 = int(L[2].pos[f0]), int(L[2].pos[f1])
        l0 = LevelStorage(L[0].spec, pos=[0, s1 - s0], crd=crd0[s0:s1] - r0, device=dev)
        l1 = LevelStorage(L[1].spec, pos=L[1].pos[s0:s1 + 1] - f0, crd=L[1].crd[f0:f1], device=dev)
        l2 = LevelStorage(L[2].spec, pos=L[2].pos[f0:f1 + 1] - e0, crd=L[2].crd[e0:e1], device=dev)
        return TensorStorage(st.format, dims, [l0, l1, l2], st.vals[e0:e1])
    if fmt_class == "ell":
        S, n = L[0].n, st.dims[0]
        crd = L[2].crd.view(S, n)[:, r0:r1].reshape(-1).contiguous() if S else L[2].crd[:0]
        vals = st.vals[:S * n].view(S, n)[:, r0:r1].reshape(-1).contiguous() if S else st.vals[:0]
        return TensorStorage(st.format, dims, [LevelStorage(L[0].spec, n=S, device=dev),
                                               LevelStorage(L[1].spec, n=r1 - r0, device=dev),
                                               LevelStorage(L[2].spec, crd=crd, device=dev)], vals)
    if fmt_class == "dia":
        # row i of the block is global row r0 + i: a diagonal at offset o
        # pairs it with column r0 + i + o, so the block is a DIA of
        # (r1 - r0) x ncols with offsets o + r0 over the same stored values
        D, n = L[0].n, st.dims[0]
        offs = L[1].offset.to(torch.int64)
        vals = st.vals[:D * n].view(D, n)[:, r0:r1].reshape(-1).contiguous()
        noffs = (offs + r0).to(torch.int32)
        l1 = LevelStorage(L[1].spec, n=r1 - r0, m=st.dims[1], offset=noffs, device=dev)
        l2 = LevelStorage(L[2].spec, offset=l1.offset, range_n=r1 - r0, device=dev)
        l2.offset = l1.offset
        out = TensorStorage(st.format, dims, [LevelStorage(L[0].spec, n=D, device=dev), l1, l2],
                            vals)
        out._host_offsets = noffs.cpu().numpy()
        return out
    raise ValueError(f"no row sharding for {fmt_class}")


_SHARDED = {"spmv": ("A",), "spmm": ("A",), "add": ("A", "B"), "mttkrp": ("X",),
            "ttv": ("X",), "ttm": ("X",)}


def _p2p_spmv_gather(A_loc, x, n, r0, r1, group):
    """SpMV of this rank's CSR row block with the all-gather fused into the
    kernel: the full y lives in symmetric memory (one buffer per rank, mapped
    into every peer), the kernel stores each row into every rank's buffer
    over NVLink (sl_spmv_csr_peers_f64), and a device-side barrier of the
    symmetric-memory handle orders the stores before anyone reads y."""
    import torch
    import torch.distributed as dist

    from . import kernels as K
    from .errors import DeviceError

    try:
        import torch.distributed._symmetric_memory as symm
    except Exception as e:                       # pragma: no cover - torch without it
        raise DeviceError(f"symmetric memory unavailable: {e}")
    dev = A_loc.vals.device
    grp = group or dist.group.WORLD
    full = symm.empty(n, dtype=torch.float64, device=dev)
    handle = symm.rendezvous(full, grp)
    world = dist.get_world_size(grp)
    ptrs = [int(handle.buffer_ptrs[q]) + 8 * r0 for q in range(world)]
    lv = A_loc.levels[1]
    K.spmv_csr_peers(r1 - r0, A_loc.dims[1], lv.pos, lv.crd, A_loc.vals, x.vals, ptrs)
    handle.barrier()
    return full


def evaluate_sharded(expr, inputs: Dict[str, "object"], out_format=None, *, group=None,
                     gather="nccl", local_eval: Optional[Callable] = None):
    """Multi-GPU `evaluate`, one process per GPU.

    Every rank passes the same global operands, resident on its device.  The
    output's first mode is cut into contiguous nnz-balanced blocks, one per
    rank; the sharded operand (the matrix / tensor whose first mode is the
    output's) is sliced on the device, the replicated ones (x, B, C, v, U —
    replicate them with `replicate` first if only one rank holds them) are
    used whole, and the rank evaluates its block with the single-GPU
    `evaluate` (no exchange during compute).  gather="nccl" (or True) all-
    gathers the blocks (dense: padded row blocks; CSR / COO: nnz totals first,
    then the arrays), so every rank returns the full result; gather="p2p"
    fuses the all-gather of a CSR SpMV's y into the kernel (each rank stores
    its rows into every rank's symmetric-memory buffer; other patterns use
    the NCCL gather); gather=False returns (local block, (r0, r1)).
    `local_eval` replaces the per-rank evaluation (tests inject the CPU oracle
    on gloo ranks)."""
    import torch

    from . import engine as E
    from .formats import TensorStorage, preset
    from .levels import LevelStorage

    rank, world = _world(group)
    p = E.plan_expression(expr, inputs, out_format)
    ev = local_eval or E.evaluate
    if p.pattern not in _SHARDED or world == 1:
        res = ev(expr, inputs, out_format)
        return res if gather else (res, (0, res.dims[0] if res.dims else 0))
    roles = _SHARDED[p.pattern]
    lead = inputs[p.operands[roles[0]]]
    n = lead.dims[0]
    bounds = row_blocks(lead, E.format_class(lead.format), world, n)
    r0, r1 = bounds[rank], bounds[rank + 1]
    local = dict(inputs)
    for role in roles:
        name = p.operands[role]
        local[name] = shard_storage(inputs[name], E.format_class(inputs[name].format), r0, r1)
    if gather == "p2p" and p.kernel == "spmv_csr" and local_eval is None and \
            inputs[p.operands["A"]].format.levels[1].props.unique and \
            E.format_class(p.out_format) == "dense1":
        full = _p2p_spmv_gather(local[p.operands["A"]], inputs[p.operands["x"]], n, r0, r1, group)
        f = p.out_format
        return TensorStorage(f, (n,), [LevelStorage(f.levels[0], n=n, device=full.device)], full)
    res = ev(expr, local, out_format)
    if not gather:
        return res, (r0, r1)
    ocls = E.format_class(res.format)
    f = res.format
    dev = res.vals.device
    if ocls.startswith("dense"):
        inner = int(np.prod(res.dims[1:])) if len(res.dims) > 1 else 1
        full = gather_row_blocks(res.vals[:(r1 - r0) * inner], [b * inner for b in bounds], group)
        dims = (n,) + tuple(res.dims[1:])
        return TensorStorage(f, dims, [LevelStorage(spec, n=d, device=dev)
                                       for spec, d in zip(f.levels, dims)], full)
    if ocls in ("csr", "coo"):
        if ocls == "csr":
            pos_l, crd_l = res.levels[1].pos, res.levels[1].crd
        else:                                   # COO block: rows back to a pointer
            rows_l = res.levels[0].crd.to(torch.int64)
            cnt = torch.bincount(rows_l, minlength=r1 - r0)
            pos_l = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev),
                               torch.cumsum(cnt, 0)]).to(torch.int32)
            crd_l = res.levels[1].crd
        nnz = int(pos_l[-1])
        pos, crd, vals = concat_csr_blocks(pos_l, crd_l[:nnz], res.vals[:nnz], group)
        if ocls == "csr":
            return TensorStorage(f, (n,) + tuple(res.dims[1:]),
                                 [LevelStorage(f.levels[0], n=n, device=dev),
                                  LevelStorage(f.levels[1], pos=pos, crd=crd, device=dev)], vals)
        rows = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device=dev),
                                       (pos[1:] - pos[:-1]).to(torch.int64))
        nz = int(crd.numel())
        return TensorStorage(f, (n,) + tuple(res.dims[1:]),
                             [LevelStorage(f.levels[0], pos=[0, nz], crd=rows, device=dev),
                              LevelStorage(f.levels[1], crd=crd, device=dev)], vals)
    raise ValueError(f"gather of a {ocls} output is not supported; use gather=False")
