"""Torch-facing API over the C ABI.  PyTorch supplies device memory, streams
and process groups; every step of the SpGEMM runs in libspgemm.so kernels.

    C = spgemm(A, B, sorted=True)          # Gustavson hash SpGEMM, two phases
    offs = rows_to_parts(A, B, nparts)      # RowsToThreads on the GPU (a8)
    t = triangle_count(L, U, G)             # L*U, mask by G, sum/2 (a9)
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class DeviceCSR:
    """CSR on a CUDA device: row_ptr int64[nrows+1] (row_ptr[0] may be > 0 for
    a row-range view), col int32, val float64 (may be None)."""
    nrows: int
    ncols: int
    row_ptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor | None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1].item() - self.row_ptr[0].item())

    def rows(self, r0: int, r1: int) -> "DeviceCSR":
        """Zero-copy row-range view [r0, r1)."""
        return DeviceCSR(r1 - r0, self.ncols, self.row_ptr[r0:r1 + 1], self.col, self.val)

    def c(self) -> _lib.spg_csr:
        assert self.row_ptr.dtype == torch.int64 and self.row_ptr.is_contiguous()
        assert self.col.dtype == torch.int32 and self.col.is_contiguous()
        if self.val is not None:
            assert self.val.dtype == torch.float64 and self.val.is_contiguous()
        return _lib.spg_csr(self.nrows, self.ncols, self.row_ptr.data_ptr(),
                            self.col.data_ptr() if self.col.numel() else 0,
                            self.val.data_ptr() if (self.val is not None and self.val.numel()) else 0)

    @staticmethod
    def from_host(M, device="cuda", non_blocking: bool = False) -> "DeviceCSR":
        """Copy a host CSR (synth.CSR-like: nrows, ncols, row_ptr, col, val)."""
        dev = torch.device(device)
        return DeviceCSR(int(M.nrows), int(M.ncols),
                         torch.as_tensor(np.ascontiguousarray(M.row_ptr, np.int64)).to(dev, non_blocking=non_blocking),
                         torch.as_tensor(np.ascontiguousarray(M.col, np.int32)).to(dev, non_blocking=non_blocking),
                         torch.as_tensor(np.ascontiguousarray(M.val, np.float64)).to(dev, non_blocking=non_blocking))

    def to_host(self):
        rp = self.row_ptr.cpu().numpy()
        rp = rp - rp[0]
        s = int(self.row_ptr[0].item())
        col = self.col[s:s + int(rp[-1])].cpu().numpy()
        val = self.val[s:s + int(rp[-1])].cpu().numpy() if self.val is not None else None
        return rp, col, val


class Context:
    """One spg_ctx (plan + grow-only workspace) bound to a CUDA device."""

    def __init__(self, device=None, allocator: str = "cuda"):
        """allocator: where the grow-only ctx workspace comes from.
        "cuda" (default) = cudaMalloc / cudaFree inside the library;
        "torch" = the PyTorch caching allocator through the C ABI's
        spg_alloc_fn / spg_free_fn callbacks (called only when the workspace
        grows).  The free callback synchronises the device first, as cudaFree
        does: a released buffer may still be read by kernels on the ctx's
        internal streams."""
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.allocator = allocator
        self._live = {}            # ptr -> bytes held through the callbacks ("torch" only)
        self._cb = (None, None)
        if allocator == "torch":
            dev = self.device.index
            live = self._live      # (the callbacks close over this dict, not over self)

            def _alloc(nbytes, stream, _user):
                try:
                    p = torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0))
                except Exception:   # (OOM: the library reports SPG_ERR_WORKSPACE)
                    return None
                live[p] = int(nbytes)
                return p

            def _free(ptr, _stream, _user):
                if ptr:
                    torch.cuda.synchronize(dev)
                    live.pop(ptr, None)
                    torch.cuda.caching_allocator_delete(ptr)

            self._cb = (_lib.ALLOC_FN(_alloc), _lib.FREE_FN(_free))
        elif allocator != "cuda":
            raise ValueError("allocator must be 'cuda' or 'torch'")
        with torch.cuda.device(self.device):
            self.handle = _lib.spg_ctx_create(*self._cb)

    @property
    def workspace_bytes(self) -> int:
        """Bytes of ctx workspace currently held through the allocator callbacks."""
        return sum(self._live.values())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.spg_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None

    def set_accumulator(self, accum: str = "auto", collision_factor: float = 1.3,
                        heap_cost: float = 8.0) -> None:
        """Sorted-output accumulator: "auto" (cost model Eq:heap_est vs
        Eq:hash_est per row, heap steps weighted by heap_cost),
        "hash" or "heap" (§4.2.3)."""
        _lib.spg_set_accumulator(self.handle, accum, collision_factor, heap_cost)

    @property
    def launches(self) -> int:
        return _lib.spg_launch_count(self.handle)

    def info(self) -> dict:
        return _lib.spg_get_info(self.handle)


_tls = threading.local()


def default_context(device=None) -> Context:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if dev not in cache:
        cache[dev] = Context(dev)
    return cache[dev]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def spg_symbolic(A: DeviceCSR, B: DeviceCSR, ctx: Context | None = None):
    """Phase 1: returns (C_row_ptr tensor, nnz(C), flop)."""
    ctx = ctx or default_context()
    rp = torch.empty(A.nrows + 1, dtype=torch.int64, device=A.row_ptr.device)
    nnz, flop = _lib.spg_symbolic(ctx.handle, A.c(), B.c(), rp.data_ptr(), _stream())
    return rp, nnz, flop


def spg_numeric(A: DeviceCSR, B: DeviceCSR, C_row_ptr: torch.Tensor, nnz: int,
                sorted: bool = True, ctx: Context | None = None,
                out: tuple | None = None) -> DeviceCSR:
    """Phase 2: allocates C.col/C.val (torch caching allocator) unless `out`
    gives them, and fills them."""
    ctx = ctx or default_context()
    dev = A.row_ptr.device
    if out is None:
        col = torch.empty(nnz, dtype=torch.int32, device=dev)
        val = torch.empty(nnz, dtype=torch.float64, device=dev)
    else:
        col, val = out
    _lib.spg_numeric(ctx.handle, A.c(), B.c(), C_row_ptr.data_ptr(),
                     col.data_ptr() if nnz else 0, val.data_ptr() if nnz else 0, sorted, _stream())
    return DeviceCSR(A.nrows, B.ncols, C_row_ptr, col, val)


def spgemm_onephase(A: DeviceCSR, B: DeviceCSR, sorted: bool = True,
                    ctx: Context | None = None) -> DeviceCSR:
    """C = A*B in ONE phase (tables sized by flop, no symbolic pass, one host
    round trip).  Raises SpgError (OVERFLOW) for rows
    with flop_i >= 8192 -- use spgemm() for those."""
    ctx = ctx or default_context()
    dev = A.row_ptr.device
    rp = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev)
    nnz, _ = _lib.spg_onephase(ctx.handle, A.c(), B.c(), rp.data_ptr(), sorted, _stream())
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.spg_onephase_emit(ctx.handle, col.data_ptr() if nnz else 0, val.data_ptr() if nnz else 0,
                           _stream())
    return DeviceCSR(A.nrows, B.ncols, rp, col, val)


def spgemm(A: DeviceCSR, B: DeviceCSR, sorted: bool = True,
           ctx: Context | None = None, method: str = "two_phase") -> DeviceCSR:
    """C = A*B (Gustavson, hash accumulator): method "two_phase"
    (symbolic + numeric) or "one_phase" (spgemm_onephase)."""
    if A.ncols != B.nrows:
        raise ValueError(f"dimension mismatch: A is {A.nrows}x{A.ncols}, B is {B.nrows}x{B.ncols}")
    ctx = ctx or default_context()
    if method == "one_phase":
        return spgemm_onephase(A, B, sorted, ctx)
    if method != "two_phase":
        raise ValueError(f"unknown method {method!r}")
    rp, nnz, _ = spg_symbolic(A, B, ctx)
    return spg_numeric(A, B, rp, nnz, sorted, ctx)


def plan_export(ctx: Context | None = None, m: int | None = None):
    """(flop[m], paper table size[m]) of the last symbolic on ctx."""
    ctx = ctx or default_context()
    m = ctx.info()["nrows"] if m is None else m
    f = torch.empty(m, dtype=torch.int64, device=ctx.device)
    t = torch.empty(m, dtype=torch.int64, device=ctx.device)
    if m:
        _lib.spg_plan_export(ctx.handle, f.data_ptr(), t.data_ptr(), _stream())
    return f, t


def rows_to_parts(A: DeviceCSR, B: DeviceCSR, nparts: int, ctx: Context | None = None):
    """offset[0..nparts] of Fig:load_balance computed on the GPU; and total flop."""
    ctx = ctx or default_context()
    return _lib.spg_rows_to_parts(ctx.handle, A.c(), B.c(), nparts, _stream())


def rows_to_parts_bytes(A: DeviceCSR, B: DeviceCSR, row_nnz: torch.Tensor, nparts: int,
                        ctx: Context | None = None):
    """Bytes-balanced split: RowsToThreads on w_i = 16 + 12
    (nnz(a_i) + flop_i + nnz(c_i)), computed on the GPU; (offsets, total)."""
    ctx = ctx or default_context()
    return _lib.spg_rows_to_parts_bytes(ctx.handle, A.c(), B.c(),
                                        row_nnz.data_ptr() if row_nnz.numel() else 0, nparts,
                                        _stream())


def mask_sum(C: DeviceCSR, G: DeviceCSR, g_row_begin: int = 0, ctx: Context | None = None) -> int:
    ctx = ctx or default_context()
    return _lib.spg_mask_sum(ctx.handle, C.c(), G.c(), g_row_begin, _stream())


def masked_sum(A: DeviceCSR, B: DeviceCSR, G: DeviceCSR, g_row_begin: int = 0,
               ctx: Context | None = None) -> float:
    """sum over (i,j) in pattern(G) of (A*B)(i,j), without forming A*B
    (fused mask)."""
    ctx = ctx or default_context()
    return _lib.spg_masked_sum(ctx.handle, A.c(), B.c(), G.c(), g_row_begin, _stream())


def masked_sum_int(A: DeviceCSR, B: DeviceCSR, G: DeviceCSR, g_row_begin: int = 0,
                   ctx: Context | None = None) -> int:
    """The same sum reduced exactly in int64 (integer-valued inputs, e.g. the
    triangle count's L*U with values 1.0); raises SpgError (OVERFLOW) if the
    inputs are not integer-valued."""
    ctx = ctx or default_context()
    return _lib.spg_masked_sum_int(ctx.handle, A.c(), B.c(), G.c(), g_row_begin, _stream())


def triangle_count_fused(L: DeviceCSR, U: DeviceCSR, G: DeviceCSR,
                         ctx: Context | None = None) -> int:
    """Triangles = sum(L*U o G)/2 with the mask fused into the product (C is
    never formed), reduced in int64; values must be integers (BASELINE
    config 5: 1.0)."""
    t = masked_sum_int(L, U, G, 0, ctx)
    if t % 2:
        raise RuntimeError(f"masked sum {t} is odd: G is not symmetric")
    return t // 2


def degree_relabel(G: DeviceCSR, ctx: Context | None = None):
    """Degree-ascending relabelling of a symmetric pattern without diagonal
    (SURVEY §8(f) row 1): returns (perm, L', U', G') with perm[r] = old
    id of new vertex r, L'/U' the strict lower/upper triangles of P G P^T and
    G' = P G P^T (sorted rows, values 1.0).  triangle_count_fused(L', U', G')
    counts the same triangles as the natural order with far fewer products."""
    ctx = ctx or default_context()
    dev = G.row_ptr.device
    n = G.nrows
    nnz = G.nnz
    if nnz % 2:
        raise ValueError("nnz(G) is odd: G is not a symmetric pattern")
    h = nnz // 2

    def out(rows, k):
        return DeviceCSR(rows, n, torch.empty(rows + 1, dtype=torch.int64, device=dev),
                         torch.empty(k, dtype=torch.int32, device=dev),
                         torch.empty(k, dtype=torch.float64, device=dev))
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    L, U, Gn = out(n, h), out(n, h), out(n, nnz)

    def ptrs(M):
        return (M.row_ptr.data_ptr(), M.col.data_ptr() if M.col.numel() else 0,
                M.val.data_ptr() if M.val.numel() else 0)
    _lib.spg_degree_relabel(ctx.handle, G.c(), perm.data_ptr() if n else 0, ptrs(L), ptrs(U),
                            ptrs(Gn), _stream())
    return perm, L, U, Gn


def triangle_count_graph(G: DeviceCSR, degree_order: bool = True, fused: bool = True,
                         ctx: Context | None = None) -> int:
    """Triangles of the undirected graph with symmetric pattern G (no
    diagonal): split G = L + U (after the degree-ascending reordering of
    P:604 when degree_order), then sum(L*U o G)/2 (fused mask, or with C
    formed in row blocks)."""
    ctx = ctx or default_context()
    if degree_order:
        _, L, U, G = degree_relabel(G, ctx)
    else:
        raise ValueError("natural order needs L and U: use triangle_count(L, U, G)")
    return triangle_count_fused(L, U, G, ctx) if fused else triangle_count(L, U, G, ctx=ctx)


def probe_stats(A: DeviceCSR, B: DeviceCSR, ctx: Context | None = None) -> dict:
    """Measured collision factor c (Eq:hash_est P:362) of the warp-tier numeric
    tables: {mode: (probes, products, keys, c = probes / products)} for
    linear probing on high / low hash bits and 4-slot chunks (SURVEY §8(f)
    row 2).  Runs the symbolic phase first (for nnz(c_i))."""
    ctx = ctx or default_context()
    rp, _, _ = spg_symbolic(A, B, ctx)
    o = _lib.spg_probe_stats(ctx.handle, A.c(), B.c(), rp.data_ptr(), _stream())
    names = ("linear_high_bits", "linear_low_bits", "chunk4_high_bits", "bucket32_warp")
    return {n: (o[3 * m], o[3 * m + 1], o[3 * m + 2], o[3 * m] / max(o[3 * m + 1], 1))
            for m, n in enumerate(names)}


def validate(M: DeviceCSR, check_sorted: bool = False, ctx: Context | None = None) -> None:
    ctx = ctx or default_context()
    _lib.spg_validate(ctx.handle, M.c(), check_sorted, _stream())


def row_blocks_by_bytes(A: DeviceCSR, B: DeviceCSR, budget_entries: int,
                        ctx: Context | None = None) -> list[int]:
    """Row offsets of blocks whose C holds at most ~budget_entries entries,
    bounded through flop (nnz(c_i) <= flop_i): RowsToThreads with enough parts."""
    ctx = ctx or default_context()
    _, tot = rows_to_parts(A, B, 1, ctx)
    nparts = max(1, -(-tot // max(1, budget_entries)))
    offs, _ = rows_to_parts(A, B, nparts, ctx)
    out = [offs[0]]
    for o in offs[1:]:
        if o != out[-1]:
            out.append(o)
    if out[-1] != A.nrows:
        out.append(A.nrows)
    return out


def triangle_count_rows(L: DeviceCSR, U: DeviceCSR, G: DeviceCSR, r0: int, r1: int,
                        sorted: bool = False, block_entries: int | None = None,
                        ctx: Context | None = None, g_shift: int = 0) -> int:
    """sum(C o G) over rows [r0, r1) of C = L*U, produced and consumed in row
    blocks (row-range views of L) so C never has to fit whole in HBM.  Row i
    of L is row g_shift + i of G (a row-scattered L block)."""
    ctx = ctx or default_context()
    if r1 <= r0:
        return 0
    Lr = L.rows(r0, r1)
    if block_entries is None:
        dev = L.row_ptr.device
        free, _ = torch.cuda.mem_get_info(dev)
        # memory cached by torch's allocator is reusable for the C blocks too
        free += torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
        block_entries = max(1 << 20, int(free * 0.6) // 12)
    offs = row_blocks_by_bytes(Lr, U, block_entries, ctx)
    total = 0
    for b0, b1 in zip(offs[:-1], offs[1:]):
        C = spgemm(Lr.rows(b0, b1), U, sorted, ctx)
        total += mask_sum(C, G, g_shift + r0 + b0, ctx)
        del C
    return total


def triangle_count(L: DeviceCSR, U: DeviceCSR, G: DeviceCSR, sorted: bool = False,
                   block_entries: int | None = None, ctx: Context | None = None) -> int:
    """Triangles = sum(C o G)/2, C = L*U (Sec 5.6, BASELINE config 5)."""
    total = triangle_count_rows(L, U, G, 0, L.nrows, sorted, block_entries, ctx)
    if total % 2:
        raise RuntimeError("sum(C o G) is odd: G is not symmetric")
    return total // 2
