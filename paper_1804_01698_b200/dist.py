"""Multi-GPU SpGEMM: one process per GPU (torch.distributed, NCCL over NVLink).

Rows of C are independent (§2: "each row of C can be
constructed independently"), so the product shards by rows of A:

1. the flop-balanced row split of A (RowsToThreads, Fig:load_balance
   P:251-270, tnum = world size) is computed on the GPU;
2. inputs are distributed from rank 0 (``distribute``): B is broadcast (its
   row_ptr first, then col / val asynchronously -- the flop pass needs only
   B.row_ptr), A (and a triangle count's mask G) are ROW-SCATTERED: each rank
   receives only its row block;
3. each rank multiplies its row block by B -> its C row block with a local
   row_ptr; optionally (``balance="bytes"``) the numeric phase runs on a split
   balanced by the minimal-bytes model instead of flop (flop
   balance leaves nnz(C) per rank uneven), using the row nnz all-gathered
   from the first symbolic pass;
4. all_gather of one int64 per rank (nnz of each block) gives every rank the
   global offsets of the blocks, so C is the concatenation of the blocks.

The local multiply, the partitions and the row-nnz pass are injectable so
the host logic is tested on CPU processes with the gloo backend; the
defaults are the CUDA path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

from .api import (Context, DeviceCSR, default_context, rows_to_parts, rows_to_parts_bytes,
                  spg_symbolic, spgemm)


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


def broadcast_csr(M, src: int = 0, device=None, group=None, async_values: bool = False):
    """Broadcast a CSR matrix from `src` (a DeviceCSR there, None elsewhere).
    With async_values the col / val broadcasts are left in flight: returns
    (matrix, [work handles]) -- row_ptr is complete on return."""
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
    works = []
    if nz:
        works.append(dist.broadcast(out.col, src, group=group, async_op=async_values))
        if hv:
            works.append(dist.broadcast(out.val, src, group=group, async_op=async_values))
    if not async_values:
        return out
    return out, [w for w in works if w is not None]


def scatter_rows(M, offsets: list, src: int = 0, device=None, group=None):
    """Row-scatter of a CSR matrix held by `src`: rank r receives rows
    [offsets[r], offsets[r+1]) with a local row_ptr (starting at 0), the
    same ncols.  Point-to-point sends from `src` (NCCL / gloo)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = device or (M.row_ptr.device if M is not None else torch.device("cuda"))
    r0, r1 = offsets[rank], offsets[rank + 1]
    meta = torch.zeros(2, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor([M.ncols, 1 if M.val is not None else 0], dtype=torch.int64)
    dist.broadcast(meta, src, group=group)
    ncols, hv = (int(x) for x in meta.tolist())
    if rank == src:
        rp_all = M.row_ptr
        for r in range(world):
            if r == src:
                continue
            a, b = offsets[r], offsets[r + 1]
            s0, s1 = int(rp_all[a].item()), int(rp_all[b].item())
            hdr = torch.tensor([s1 - s0], dtype=torch.int64, device=device)
            dist.send(hdr, r, group=group)
            dist.send((rp_all[a:b + 1] - s0).contiguous(), r, group=group)
            if s1 > s0:
                dist.send(M.col[s0:s1].contiguous(), r, group=group)
                if hv:
                    dist.send(M.val[s0:s1].contiguous(), r, group=group)
        s0, s1 = int(rp_all[r0].item()), int(rp_all[r1].item())
        return DeviceCSR(r1 - r0, ncols, (rp_all[r0:r1 + 1] - s0).contiguous(),
                         M.col[s0:s1].contiguous(),
                         M.val[s0:s1].contiguous() if hv else None)
    hdr = torch.zeros(1, dtype=torch.int64, device=device)
    dist.recv(hdr, src, group=group)
    nz = int(hdr.item())
    rp = torch.empty(r1 - r0 + 1, dtype=torch.int64, device=device)
    dist.recv(rp, src, group=group)
    col = torch.empty(nz, dtype=torch.int32, device=device)
    val = torch.empty(nz, dtype=torch.float64, device=device) if hv else None
    if nz:
        dist.recv(col, src, group=group)
        if hv:
            dist.recv(val, src, group=group)
    return DeviceCSR(r1 - r0, ncols, rp, col, val)


def distribute(A, B, G=None, src: int = 0, device=None, group=None, partition: Callable | None = None,
               ctx: Context | None = None):
    """Inputs held by rank `src` (None elsewhere) -> every rank's share:
    the flop-balanced offsets (computed on `src`'s GPU, broadcast), this
    rank's row block of A (and of G, the triangle mask), and all of B.  B's
    col / val broadcasts run asynchronously while A is scattered.  Returns
    (A_block, B, G_block or None, offsets)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = device or torch.device("cuda", torch.cuda.current_device())
    Bl, works = broadcast_csr(B if rank == src else None, src, device, group, async_values=True)
    offs_t = torch.zeros(world + 1, dtype=torch.int64, device=device)
    if rank == src:
        offs, _ = (partition or (lambda X, Y, n: rows_to_parts(X, Y, n, ctx)))(A, Bl, world)
        offs_t[:] = torch.tensor(offs, dtype=torch.int64)
    dist.broadcast(offs_t, src, group=group)
    offs = [int(x) for x in offs_t.tolist()]
    Al = scatter_rows(A if rank == src else None, offs, src, device, group)
    has_g = _flag(G is not None, rank, src, device, group)
    Gl = scatter_rows(G if rank == src else None, offs, src, device, group) if has_g else None
    for w in works:
        w.wait()
    return Al, Bl, Gl, offs


def _flag(v: bool, rank: int, src: int, device, group) -> bool:
    """Broadcast a boolean from src (whether an optional matrix exists)."""
    t = torch.tensor([1 if (v and rank == src) else 0], dtype=torch.int64, device=device)
    dist.broadcast(t, src, group=group)
    return bool(t.item())


def partition_rows(A, B, nparts: int, ctx: Context | None = None) -> tuple[list[int], int]:
    """Flop-balanced contiguous row split (Fig:load_balance) computed on the GPU."""
    return rows_to_parts(A, B, nparts, ctx or default_context())


def _allgather_cat(x: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenation (in rank order) of 1-D int64 tensors of different lengths."""
    world = dist.get_world_size(group)
    n = torch.tensor([x.numel()], dtype=torch.int64, device=x.device)
    ns = [torch.zeros(1, dtype=torch.int64, device=x.device) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(ns) if ns else 0
    pad = torch.zeros(mx, dtype=x.dtype, device=x.device)
    pad[:x.numel()] = x
    outs = [torch.empty(mx, dtype=x.dtype, device=x.device) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:k] for o, k in zip(outs, ns)])


def spgemm_dist(A, B, sorted: bool = True, group=None, ctx: Context | None = None,
                partition: Callable | None = None,
                local_spgemm: Callable | None = None, balance: str = "flop",
                row_nnz: Callable | None = None,
                partition_bytes: Callable | None = None) -> DistBlock:
    """C = A*B over the ranks of `group`; A and B must be present on every rank
    (replicated, e.g. broadcast_csr).  Returns this rank's block.

    balance="flop": the RowsToThreads split by flop (Fig:load_balance).
    balance="bytes": a first symbolic pass on the flop split gives nnz(c_i) of
    the rank's rows; the row counts are all-gathered and the numeric phase
    runs on the split balanced by the per-row minimal bytes;
    when that split moves a rank's rows, its symbolic phase is redone on the
    new rows (the price of the balance: it pays when the bytes imbalance of
    the flop split exceeds the symbolic share of a step)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if partition is None:
        offs, _ = partition_rows(A, B, world, ctx)
    else:
        offs, _ = partition(A, B, world)
    if balance not in ("flop", "bytes"):
        raise ValueError(f"unknown balance {balance!r}")
    if balance == "bytes" and world > 1:
        r0, r1 = offs[rank], offs[rank + 1]
        if row_nnz is None:
            rp, _, _ = spg_symbolic(A.rows(r0, r1), B, ctx)
            mine = (rp[1:] - rp[:-1]).contiguous()
        else:
            mine = row_nnz(A, B, r0, r1)
        allnnz = _allgather_cat(mine, group)
        if partition_bytes is None:
            offs2, _ = rows_to_parts_bytes(A, B, allnnz, world, ctx)
        else:
            offs2 = partition_bytes(A, B, allnnz, world)
        offs = list(offs2)
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
    fused=True sums the masked products without forming C (spg_masked_sum_int)."""
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
