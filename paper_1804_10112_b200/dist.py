"""Multi-GPU partitioning of the hot path.

SpMV and MTTKRP shard by contiguous, nnz-balanced blocks of output rows
(slices): each rank owns rows [r0, r1), computes its block of y (A) with no
data-path exchange, and reads a replicated x (B, C).  torch.distributed
over NCCL is used only to replicate x / the factors once (broadcast) and,
optionally, to gather the row blocks of y back (all-gather of padded
blocks).  One process per GPU.

The host-side partition and shard functions are pure numpy, so the
multi-rank logic is covered by world_size-2 gloo tests on CPU
(tests/test_dist_gloo.py); the kernels each rank runs are the single-GPU ones.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

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
    pad = torch.zeros(m, dtype=y_local.dtype, device=y_local.device)
    pad[:y_local.numel()] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[p][:sizes[p]] for p in range(world)])


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
