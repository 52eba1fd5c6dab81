"""ctypes binding of include/spgemm.h (argument marshalling only).

Every function here has the name of the C entry point it calls and takes
plain integers (device pointers, sizes, stream handles).  No computation
happens in Python; there is no CPU fallback: if libspgemm.so is missing or
cannot be loaded the import fails loudly.
"""
from __future__ import annotations

import ctypes as ct
import os

from .build import LIB

SPG_OK = 0
STATUS = {0: "SPG_OK", 1: "SPG_ERR_INVALID_ARG", 2: "SPG_ERR_DIM_MISMATCH",
          3: "SPG_ERR_INDEX_RANGE", 4: "SPG_ERR_OVERFLOW", 5: "SPG_ERR_WORKSPACE",
          6: "SPG_ERR_STATE", 7: "SPG_ERR_CUDA"}

# every symbol include/spgemm.h declares
EXPORTS = ("spg_ctx_create", "spg_ctx_destroy", "spg_last_error", "spg_launch_count",
           "spg_symbolic", "spg_numeric", "spg_get_info", "spg_plan_export",
           "spg_rows_to_parts", "spg_mask_sum", "spg_validate", "spg_profile_enable", "spg_set_serial_bins",
           "spg_profile_reset", "spg_profile_count", "spg_profile_record",
           "spg_debug_counters", "spg_masked_sum", "spg_degree_relabel",
           "spg_probe_stats", "spg_masked_sum_int", "spg_set_accumulator", "spg_onephase",
           "spg_onephase_emit", "spg_rows_to_parts_bytes")


class spg_csr(ct.Structure):
    _fields_ = [("nrows", ct.c_int64), ("ncols", ct.c_int64), ("row_ptr", ct.c_void_p),
                ("col_idx", ct.c_void_p), ("val", ct.c_void_p)]


class spg_info(ct.Structure):
    _fields_ = [("nrows", ct.c_int64), ("flop_total", ct.c_int64), ("nnz_total", ct.c_int64),
                ("max_row_flop", ct.c_int64), ("max_row_nnz", ct.c_int64),
                ("sym_bin_rows", ct.c_int64 * 12), ("num_bin_rows", ct.c_int64 * 12),
                ("heap_rows", ct.c_int64)]


class SpgError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load(path: str | None = None) -> ct.CDLL:
    """Load libspgemm.so (raises if it is missing: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with "
                          "`python -m paper_1804_01698_b200.build` (no CPU fallback exists)")
    lib = ct.CDLL(path)
    vp, i64, i64p = ct.c_void_p, ct.c_int64, ct.POINTER(ct.c_int64)
    csrp = ct.POINTER(spg_csr)
    lib.spg_ctx_create.argtypes = [ct.POINTER(vp), vp, vp, vp]
    lib.spg_ctx_destroy.argtypes = [vp]
    lib.spg_last_error.argtypes = [vp]
    lib.spg_last_error.restype = ct.c_char_p
    lib.spg_launch_count.argtypes = [vp]
    lib.spg_launch_count.restype = i64
    lib.spg_symbolic.argtypes = [vp, csrp, csrp, vp, i64p, i64p, vp]
    lib.spg_numeric.argtypes = [vp, csrp, csrp, vp, vp, vp, ct.c_int, vp]
    lib.spg_get_info.argtypes = [vp, ct.POINTER(spg_info)]
    lib.spg_plan_export.argtypes = [vp, vp, vp, vp]
    lib.spg_rows_to_parts.argtypes = [vp, csrp, csrp, i64, i64p, i64p, vp]
    lib.spg_mask_sum.argtypes = [vp, csrp, csrp, i64, i64p, vp]
    lib.spg_validate.argtypes = [vp, csrp, ct.c_int, vp]
    lib.spg_profile_enable.argtypes = [vp, ct.c_int]
    lib.spg_set_serial_bins.argtypes = [vp, ct.c_int]
    lib.spg_profile_reset.argtypes = [vp]
    lib.spg_profile_count.argtypes = [vp]
    lib.spg_profile_count.restype = i64
    lib.spg_profile_record.argtypes = [vp, i64, ct.POINTER(ct.c_char_p), ct.POINTER(ct.c_float)]
    lib.spg_debug_counters.argtypes = [vp, i64p, vp]
    lib.spg_masked_sum.argtypes = [vp, csrp, csrp, csrp, i64, ct.POINTER(ct.c_double), vp]
    lib.spg_masked_sum_int.argtypes = [vp, csrp, csrp, csrp, i64, i64p, vp]
    lib.spg_set_accumulator.argtypes = [vp, ct.c_int, ct.c_double, ct.c_double]
    lib.spg_onephase.argtypes = [vp, csrp, csrp, vp, i64p, i64p, ct.c_int, vp]
    lib.spg_onephase_emit.argtypes = [vp, vp, vp, vp]
    lib.spg_rows_to_parts_bytes.argtypes = [vp, csrp, csrp, vp, i64, i64p, i64p, vp]
    lib.spg_degree_relabel.argtypes = [vp, csrp] + [vp] * 11
    lib.spg_probe_stats.argtypes = [vp, csrp, csrp, vp, i64p, vp]
    for name in EXPORTS:
        if name not in ("spg_last_error", "spg_launch_count", "spg_profile_count"):
            getattr(lib, name).restype = ct.c_int
    _lib = lib
    return lib


def _check(ctx, fn: str, status: int):
    if status != SPG_OK:
        msg = load().spg_last_error(ctx).decode() if ctx else ""
        raise SpgError(fn, status, msg)


# spg_alloc_fn / spg_free_fn of include/spgemm.h
ALLOC_FN = ct.CFUNCTYPE(ct.c_void_p, ct.c_size_t, ct.c_void_p, ct.c_void_p)
FREE_FN = ct.CFUNCTYPE(None, ct.c_void_p, ct.c_void_p, ct.c_void_p)


def spg_ctx_create(alloc=None, free_fn=None) -> int:
    """alloc / free_fn: ALLOC_FN / FREE_FN instances (both or neither); the
    caller keeps them alive for the lifetime of the ctx."""
    h = ct.c_void_p()
    st = load().spg_ctx_create(ct.byref(h), alloc, free_fn, None)
    _check(None, "spg_ctx_create", st)
    return h.value


def spg_ctx_destroy(ctx: int) -> None:
    _check(None, "spg_ctx_destroy", load().spg_ctx_destroy(ctx))


def spg_launch_count(ctx: int) -> int:
    return int(load().spg_launch_count(ctx))


def spg_symbolic(ctx: int, A: spg_csr, B: spg_csr, c_row_ptr: int, stream: int):
    nnz, flop = ct.c_int64(), ct.c_int64()
    st = load().spg_symbolic(ctx, ct.byref(A), ct.byref(B), c_row_ptr, ct.byref(nnz),
                             ct.byref(flop), stream)
    _check(ctx, "spg_symbolic", st)
    return nnz.value, flop.value


def spg_numeric(ctx: int, A: spg_csr, B: spg_csr, c_row_ptr: int, c_col: int, c_val: int,
                sorted_: bool, stream: int) -> None:
    st = load().spg_numeric(ctx, ct.byref(A), ct.byref(B), c_row_ptr, c_col, c_val,
                            1 if sorted_ else 0, stream)
    _check(ctx, "spg_numeric", st)


def spg_get_info(ctx: int) -> dict:
    info = spg_info()
    _check(ctx, "spg_get_info", load().spg_get_info(ctx, ct.byref(info)))
    return {"nrows": info.nrows, "flop_total": info.flop_total, "nnz_total": info.nnz_total,
            "max_row_flop": info.max_row_flop, "max_row_nnz": info.max_row_nnz,
            "sym_bin_rows": list(info.sym_bin_rows), "num_bin_rows": list(info.num_bin_rows),
            "heap_rows": info.heap_rows}


def spg_plan_export(ctx: int, flop_out: int, tsize_out: int, stream: int) -> None:
    _check(ctx, "spg_plan_export", load().spg_plan_export(ctx, flop_out, tsize_out, stream))


def spg_rows_to_parts(ctx: int, A: spg_csr, B: spg_csr, nparts: int, stream: int):
    off = (ct.c_int64 * (nparts + 1))()
    tot = ct.c_int64()
    st = load().spg_rows_to_parts(ctx, ct.byref(A), ct.byref(B), nparts,
                                  ct.cast(off, ct.POINTER(ct.c_int64)), ct.byref(tot), stream)
    _check(ctx, "spg_rows_to_parts", st)
    return [int(x) for x in off], tot.value


def spg_mask_sum(ctx: int, C: spg_csr, G: spg_csr, g_row_begin: int, stream: int) -> int:
    s = ct.c_int64()
    st = load().spg_mask_sum(ctx, ct.byref(C), ct.byref(G), g_row_begin, ct.byref(s), stream)
    _check(ctx, "spg_mask_sum", st)
    return s.value


def spg_validate(ctx: int, M: spg_csr, check_sorted: bool, stream: int) -> None:
    st = load().spg_validate(ctx, ct.byref(M), 1 if check_sorted else 0, stream)
    _check(ctx, "spg_validate", st)


def spg_profile_enable(ctx: int, enable: bool) -> None:
    _check(ctx, "spg_profile_enable", load().spg_profile_enable(ctx, 1 if enable else 0))


def spg_set_serial_bins(ctx: int, on: bool) -> None:
    _check(ctx, "spg_set_serial_bins", load().spg_set_serial_bins(ctx, 1 if on else 0))


def spg_profile_reset(ctx: int) -> None:
    _check(ctx, "spg_profile_reset", load().spg_profile_reset(ctx))


def spg_profile_records(ctx: int) -> list[tuple[str, float]]:
    """[(kernel name, ms)] of every launch recorded since the last reset."""
    lib = load()
    n = int(lib.spg_profile_count(ctx))
    out = []
    name, ms = ct.c_char_p(), ct.c_float()
    for i in range(n):
        _check(ctx, "spg_profile_record", lib.spg_profile_record(ctx, i, ct.byref(name), ct.byref(ms)))
        out.append((name.value.decode(), float(ms.value)))
    return out


def spg_debug_counters(ctx: int, stream: int = 0) -> list[int]:
    out = (ct.c_int64 * 16)()
    _check(ctx, "spg_debug_counters", load().spg_debug_counters(ctx, out, stream))
    return list(out)


def spg_masked_sum(ctx: int, A: spg_csr, B: spg_csr, G: spg_csr, g_row_begin: int,
                   stream: int) -> float:
    out = ct.c_double(0.0)
    _check(ctx, "spg_masked_sum",
           load().spg_masked_sum(ctx, ct.byref(A), ct.byref(B), ct.byref(G), g_row_begin,
                                 ct.byref(out), stream))
    return out.value


ACCUM = {"auto": 0, "hash": 1, "heap": 2}


def spg_onephase(ctx: int, A: spg_csr, B: spg_csr, c_row_ptr: int, sorted: bool, stream: int):
    nnz, flop = ct.c_int64(0), ct.c_int64(0)
    _check(ctx, "spg_onephase", load().spg_onephase(ctx, ct.byref(A), ct.byref(B), c_row_ptr,
                                                    ct.byref(nnz), ct.byref(flop), int(sorted), stream))
    return nnz.value, flop.value


def spg_rows_to_parts_bytes(ctx: int, A: spg_csr, B: spg_csr, row_nnz: int, nparts: int,
                            stream: int):
    off = (ct.c_int64 * (nparts + 1))()
    tot = ct.c_int64()
    _check(ctx, "spg_rows_to_parts_bytes",
           load().spg_rows_to_parts_bytes(ctx, ct.byref(A), ct.byref(B), row_nnz, nparts, off,
                                          ct.byref(tot), stream))
    return list(off), tot.value


def spg_onephase_emit(ctx: int, c_col: int, c_val: int, stream: int) -> None:
    _check(ctx, "spg_onephase_emit", load().spg_onephase_emit(ctx, c_col, c_val, stream))


def spg_set_accumulator(ctx: int, accum: str = "auto", collision_factor: float = 1.3,
                        heap_cost: float = 8.0) -> None:
    _check(ctx, "spg_set_accumulator",
           load().spg_set_accumulator(ctx, ACCUM[accum], float(collision_factor), float(heap_cost)))


def spg_masked_sum_int(ctx: int, A: spg_csr, B: spg_csr, G: spg_csr, g_row_begin: int,
                       stream: int) -> int:
    out = ct.c_int64(0)
    _check(ctx, "spg_masked_sum_int",
           load().spg_masked_sum_int(ctx, ct.byref(A), ct.byref(B), ct.byref(G), g_row_begin,
                                     ct.byref(out), stream))
    return out.value


def spg_degree_relabel(ctx: int, G: spg_csr, perm: int, L: tuple, U: tuple, Gn: tuple,
                       stream: int) -> None:
    """L, U, Gn: (row_ptr, col, val) device pointers of the outputs."""
    _check(ctx, "spg_degree_relabel",
           load().spg_degree_relabel(ctx, ct.byref(G), perm, *L, *U, *Gn, stream))


def spg_probe_stats(ctx: int, A: spg_csr, B: spg_csr, c_row_ptr: int, stream: int) -> list[int]:
    out = (ct.c_int64 * 12)()
    _check(ctx, "spg_probe_stats",
           load().spg_probe_stats(ctx, ct.byref(A), ct.byref(B), c_row_ptr, out, stream))
    return list(out)
