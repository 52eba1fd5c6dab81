"""CPU oracle for the hash-SpGEMM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_1804_01698_b200`` never imports it and shares no code
with it (see DESIGN.md §"Oracle").

The arithmetic lives in ``spa_oracle.c`` (plain C, fp64, dense sparse
accumulator, -ffp-contract=off); this file only builds/loads it and marshals
numpy arrays.  Functions and the PAPER.md passages they follow:

* ``flop``            Fig:load_balance l.1-6, flop definition
* ``table_size``      Fig:hash_spgemm l.5-13
* ``rows_to_threads`` Fig:load_balance l.7-14, lowbnd P:246
* ``spgemm``          Fig:code_spgemm with a SPA; sorted
                      output
* ``mask_sum`` / ``triangle_count``  Sec 5.6 + BASELINE config 5
* ``degree_relabel``  Sec 5.6 P:604 ("we reorder rows with increasing number
                      of nonzeros ... splits the reordered matrix A as A = L + U")

Pins (tests/test_oracle.py): dense brute force, identity, stencil and K_n
closed forms, tall-skinny column identity, row-sum identity, L*U symmetry,
triangle brute force, the SPEC worked examples (tests/golden/).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = ct.POINTER(ct.c_int64)
_i32p = ct.POINTER(ct.c_int32)
_f64p = ct.POINTER(ct.c_double)


def build(force: bool = False) -> str:
    """Compile spa_oracle.c with gcc (OpenMP, -O2, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC",
               "-shared", "-o", _LIB + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ct.CDLL(_LIB)
        lib.oracle_flop.restype = ct.c_int64
        lib.oracle_flop.argtypes = [ct.c_int64, _i64p, _i32p, _i64p, _i64p]
        lib.oracle_table_size.restype = ct.c_int64
        lib.oracle_table_size.argtypes = [ct.c_int64, ct.c_int64]
        lib.oracle_rows_to_threads.restype = None
        lib.oracle_rows_to_threads.argtypes = [ct.c_int64, _i64p, ct.c_int64, _i64p]
        lib.oracle_symbolic.restype = ct.c_int
        lib.oracle_symbolic.argtypes = [ct.c_int64, _i64p, _i32p, _i64p, _i32p,
                                        ct.c_int64, ct.c_int64, _i64p, ct.c_int]
        lib.oracle_numeric.restype = ct.c_int
        lib.oracle_numeric.argtypes = [ct.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p,
                                       _f64p, ct.c_int64, ct.c_int64, _i64p, _i32p,
                                       _f64p, ct.c_int]
        lib.oracle_mask_sum.restype = ct.c_int64
        lib.oracle_mask_sum.argtypes = [ct.c_int64, ct.c_int64, _i64p, _i32p, _f64p,
                                        _i64p, _i32p]
        _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def flop(A, B) -> tuple[np.ndarray, int]:
    """Per-row flop of C = A*B and the total."""
    assert A.ncols == B.nrows
    lib = _load()
    out = np.zeros(A.nrows, dtype=np.int64)
    arp, acol, brp = _c(A.row_ptr, np.int64), _c(A.col, np.int32), _c(B.row_ptr, np.int64)
    tot = lib.oracle_flop(A.nrows, _p(arp, _i64p), _p(acol, _i32p), _p(brp, _i64p),
                          _p(out, _i64p))
    return out, int(tot)


def table_size(flop_i: int, ncols: int) -> int:
    """Lowest 2^n strictly greater than min(N_col, flop)."""
    return int(_load().oracle_table_size(int(flop_i), int(ncols)))


def rows_to_threads(flop_rows: np.ndarray, tnum: int) -> np.ndarray:
    """offset[0..tnum] of Fig:load_balance from per-row flop."""
    m = len(flop_rows)
    ps = np.zeros(m + 1, dtype=np.int64)
    ps[1:] = np.cumsum(np.asarray(flop_rows, dtype=np.int64))  # ParallelPrefixSum
    off = np.zeros(tnum + 1, dtype=np.int64)
    _load().oracle_rows_to_threads(m, _p(ps, _i64p), tnum, _p(off, _i64p))
    return off


def spgemm(A, B, row_begin: int = 0, row_end: int | None = None,
           nthreads: int = 0):
    """Rows [row_begin, row_end) of C = A*B, sorted columns.

    Returns (row_ptr int64[r+1] starting at 0, col int32, val float64)."""
    assert A.ncols == B.nrows, "dimension mismatch"
    lib = _load()
    if row_end is None:
        row_end = A.nrows
    r = row_end - row_begin
    arp, acol, aval = _c(A.row_ptr, np.int64), _c(A.col, np.int32), _c(A.val, np.float64)
    brp, bcol, bval = _c(B.row_ptr, np.int64), _c(B.col, np.int32), _c(B.val, np.float64)
    nnz = np.zeros(max(r, 0), dtype=np.int64)
    if r > 0:
        rc = lib.oracle_symbolic(B.ncols, _p(arp, _i64p), _p(acol, _i32p), _p(brp, _i64p),
                                 _p(bcol, _i32p), row_begin, row_end, _p(nnz, _i64p),
                                 nthreads)
        if rc != 0:
            raise MemoryError("oracle_symbolic failed")
    rp = np.zeros(max(r, 0) + 1, dtype=np.int64)
    np.cumsum(nnz, out=rp[1:])
    col = np.zeros(int(rp[-1]), dtype=np.int32)
    val = np.zeros(int(rp[-1]), dtype=np.float64)
    if r > 0:
        rc = lib.oracle_numeric(B.ncols, _p(arp, _i64p), _p(acol, _i32p), _p(aval, _f64p),
                                _p(brp, _i64p), _p(bcol, _i32p), _p(bval, _f64p),
                                row_begin, row_end, _p(rp, _i64p), _p(col, _i32p),
                                _p(val, _f64p), nthreads)
        if rc != 0:
            raise RuntimeError(f"oracle_numeric failed ({rc})")
    return rp, col, val


def row_nnz(A, B, row_begin: int = 0, row_end: int | None = None,
            nthreads: int = 0) -> np.ndarray:
    """nnz(c_i*) for rows [row_begin, row_end) (symbolic phase only)."""
    lib = _load()
    if row_end is None:
        row_end = A.nrows
    r = row_end - row_begin
    arp, acol = _c(A.row_ptr, np.int64), _c(A.col, np.int32)
    brp, bcol = _c(B.row_ptr, np.int64), _c(B.col, np.int32)
    nnz = np.zeros(max(r, 0), dtype=np.int64)
    if r > 0:
        rc = lib.oracle_symbolic(B.ncols, _p(arp, _i64p), _p(acol, _i32p), _p(brp, _i64p),
                                 _p(bcol, _i32p), row_begin, row_end, _p(nnz, _i64p),
                                 nthreads)
        if rc != 0:
            raise MemoryError("oracle_symbolic failed")
    return nnz


def mask_sum(c_rp, c_col, c_val, G, row_begin: int = 0) -> int:
    """Sum of C(i,j) over (i,j) in pattern(G) for the C row block starting at
    row_begin (c_rp local, sorted columns)."""
    lib = _load()
    r = len(c_rp) - 1
    crp, ccol, cval = _c(c_rp, np.int64), _c(c_col, np.int32), _c(c_val, np.float64)
    grp, gcol = _c(G.row_ptr, np.int64), _c(G.col, np.int32)
    return int(lib.oracle_mask_sum(row_begin, row_begin + r, _p(crp, _i64p),
                                   _p(ccol, _i32p), _p(cval, _f64p), _p(grp, _i64p),
                                   _p(gcol, _i32p)))


def triangle_count(L, U, G, block_rows: int | None = None, nthreads: int = 0) -> int:
    """Triangles = sum(C o G) / 2 with C = L*U (BASELINE config 5), computed in
    row blocks so C never has to be held whole."""
    m = L.nrows
    block_rows = block_rows or m
    total = 0
    for r0 in range(0, m, block_rows):
        r1 = min(m, r0 + block_rows)
        rp, col, val = spgemm(L, U, r0, r1, nthreads)
        total += mask_sum(rp, col, val, G, r0)
    assert total % 2 == 0, "sum(C o G) must be even for symmetric G"
    return total // 2


class OCSR:
    """Minimal CSR record returned by the oracle (row_ptr int64, col int32, val f64)."""

    def __init__(self, nrows, ncols, row_ptr, col, val):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptr, self.col, self.val = row_ptr, col, val


def degree_relabel(G):
    """Degree-ascending relabelling: new id of vertex v = rank of
    (deg(v), v) ascending; G' = P G P^T; L' / U' = strict lower / upper
    triangle of G' (the split "A = L + U" of the reordered matrix).  Rows with
    ascending columns, values 1.0.  Returns (perm, L', U', G') with perm[r] =
    old id of new vertex r."""
    n = G.nrows
    rp = np.asarray(G.row_ptr, dtype=np.int64)
    deg = np.diff(rp)
    perm = np.lexsort((np.arange(n), deg))          # by degree, then by id
    rank = np.empty(n, dtype=np.int64)
    rank[perm] = np.arange(n)
    old_rows = np.repeat(np.arange(n), deg)
    r2 = rank[old_rows]
    c2 = rank[np.asarray(G.col[rp[0]:rp[-1]], dtype=np.int64)]
    order = np.lexsort((c2, r2))                    # row-major, ascending columns
    r2, c2 = r2[order], c2[order]

    def csr(keep):
        rr, cc = r2[keep], c2[keep]
        ptr = np.zeros(n + 1, dtype=np.int64)
        ptr[1:] = np.cumsum(np.bincount(rr, minlength=n))
        return OCSR(n, n, ptr, cc.astype(np.int32), np.ones(len(cc)))
    return (perm.astype(np.int32), csr(c2 < r2), csr(c2 > r2), csr(np.ones(len(r2), bool)))
