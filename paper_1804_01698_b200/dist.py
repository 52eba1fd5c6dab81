"""Multi-GPU SpGEMM: one process per GPU (torch.distributed, NCCL over NVLink).

Rows of C are independent (§2: "each row of C can be
constructed independently"), so the product shards by rows of A:

1. rank 0 holds A and B; B (and A) are broadcast once (NCCL broadcast over
   NVLink/NVSwitch) -- the only data exchange of the path;
2. every rank computes the same flop-balanced row split of A on its GPU
   (RowsToThreads, Fig:load_balance P:251-270, with tnum = world size);
3. each rank multiplies its row-range VIEW of A (no copy) by B -> its C row
   block with a local row_ptr;
4. all_gather of one int64 per rank (nnz of each block) gives every rank the
   global offsets of the blocks, so C is the concatenation of the blocks.

The local multiply is injectable (`local_spgemm`) so the host logic can be
tested on CPU processes with the gloo backend; the default is the CUDA path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

from .api import Context, DeviceCSR, default_context, rows_to_parts, spgemm


@dataclass
class DistBlock:
    """This rank's block of C = A*B: rows [row_begin, row_end) of C, stored as
    a DeviceCSR with local row_ptr (starting at 0); nnz_offset = number of C
    entries in the blocks of lower ranks; nnz_total = nnz(C)."""
    C: object
    row_begin: int
    row_end: int
    nnz_offset: int
    nnz_total: int
    offsets: list


def broadcast_csr(M, src: int = 0, device=None, group=None):
    """Broadcast a CSR matrix from `src` (a DeviceCSR there, None elsewhere)."""
    rank = dist.get_rank(group)
    device = device or (M.row_ptr.device if M is not None else torch.device("cuda"))
    meta = torch.zeros(4, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor([M.nrows, M.ncols, M.col.numel(), 1 if M.val is not None else 0],
                               dtype=torch.int64)
    dist.broadcast(meta, src, group=group)
    n, k, nz, hv = (int(x) for x in meta.tolist())
    if rank == src:
        out = M
    else:
        out = DeviceCSR(n, k, torch.empty(n + 1, dtype=torch.int64, device=device),
                        torch.empty(nz, dtype=torch.int32, device=device),
                        torch.empty(nz, dtype=torch.float64, device=device) if hv else None)
    dist.broadcast(out.row_ptr, src, group=group)
    if nz:
        dist.broadcast(out.col, src, group=group)
        if hv:
            dist.broadcast(out.val, src, group=group)
    return out


def partition_rows(A, B, nparts: int, ctx: Context | None = None) -> tuple[list[int], int]:
    """Flop-balanced contiguous row split (Fig:load_balance) computed on the GPU."""
    return rows_to_parts(A, B, nparts, ctx or default_context())


def spgemm_dist(A, B, sorted: bool = True, group=None, ctx: Context | None = None,
                partition: Callable | None = None,
                local_spgemm: Callable | None = None) -> DistBlock:
    """C = A*B over the ranks of `group`; A and B must be present on every rank
    (use broadcast_csr first).  Returns this rank's block."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if partition is None:
        offs, _ = partition_rows(A, B, world, ctx)
    else:
        offs, _ = partition(A, B, world)
    r0, r1 = offs[rank], offs[rank + 1]
    if local_spgemm is None:
        C = spgemm(A.rows(r0, r1), B, sorted, ctx)
        nnz = C.col.numel()
        dev = C.row_ptr.device
    else:
        C = local_spgemm(A, B, r0, r1, sorted)
        nnz = int(C[0][-1]) if isinstance(C, tuple) else C.col.numel()
        dev = torch.device("cpu")
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([nnz], dtype=torch.int64, device=dev), group=group)
    counts = [int(c.item()) for c in counts]
    return DistBlock(C, r0, r1, sum(counts[:rank]), sum(counts), offs)


def triangle_count_dist(L, U, G, group=None, ctx: Context | None = None,
                        fused: bool = False) -> int:
    """Triangle count of BASELINE config 5 over the ranks: each rank counts
    sum(C o G) on its flop-balanced row block of C = L*U, then all_reduce(SUM).
    fused=True sums the masked products without forming C (spg_masked_sum)."""
    from .api import masked_sum_int, triangle_count_rows
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    offs, _ = partition_rows(L, U, world, ctx)
    r0, r1 = offs[rank], offs[rank + 1]
    if fused:
        part = masked_sum_int(L.rows(r0, r1), U, G, r0, ctx) if r1 > r0 else 0
    else:
        part = triangle_count_rows(L, U, G, r0, r1, ctx=ctx)
    t = torch.tensor([part], dtype=torch.int64, device=L.row_ptr.device)
    dist.all_reduce(t, group=group)
    total = int(t.item())
    if total % 2:
        raise RuntimeError("sum(C o G) is odd: G is not symmetric")
    return total // 2


def triangle_count_graph_dist(G, group=None, ctx: Context | None = None, fused: bool = True) -> int:
    """Triangles of the graph G (replicated on every rank): every rank computes
    the same degree-ascending relabelling (deterministic), then
    triangle_count_dist on the reordered split L' + U'."""
    from .api import degree_relabel
    _, L, U, G2 = degree_relabel(G, ctx)
    return triangle_count_dist(L, U, G2, group, ctx, fused=fused)
