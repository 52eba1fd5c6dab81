"""Seeded synthetic CSR inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path (``paper_1804_01698_b200``).  It draws random matrices and nothing else:
it contains none of the SpGEMM arithmetic (no flop count, no product, no
accumulation, no sizing rule).  Every generator is deterministic in its seed
(numpy PCG64 via ``np.random.default_rng``).

Paper context (§5.1 "Input Types"): synthetic matrices come
from R-MAT with ER (a=b=c=d=.25) or G500 (a=.57, b=c=.19, d=.05) seeds; "a scale
n matrix represents 2^n-by-2^n" and the edge factor is nnz/n.  The concrete
recipes of the five BASELINE.json configs (ER Poisson rows, 27-point stencil,
R-MAT scale 20, tall-skinny frontier, triangular L/U) are documented in
DESIGN.md §"Input recipe".
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "CSR", "from_coo", "er_poisson", "stencil27", "rmat_edges", "rmat",
    "symmetrise_pattern", "frontier", "tril_strict", "triu_strict",
    "identity", "shuffle_within_rows", "with_values", "random_sparse",
    "complete_graph", "workload", "WORKLOADS",
]


@dataclass
class CSR:
    """Host CSR matrix: int64 row_ptr[nrows+1], int32 col[nnz], float64 val[nnz].

    Layout per PAPER.md §2: ``rpts`` of length n+1, ``cols`` and ``vals``
    of length nnz; row order of columns unspecified (sorted=True means every row
    is strictly increasing).
    """
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    sorted: bool = True

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1] - self.row_ptr[0]) if self.nrows >= 0 else 0

    def row(self, i: int):
        s, e = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        return self.col[s:e], self.val[s:e]

    def check(self) -> None:
        assert self.row_ptr.dtype == np.int64 and self.col.dtype == np.int32
        assert self.val.dtype == np.float64
        assert len(self.row_ptr) == self.nrows + 1
        assert len(self.col) == len(self.val) == int(self.row_ptr[-1])
        assert np.all(np.diff(self.row_ptr) >= 0)
        if len(self.col):
            assert self.col.min() >= 0 and self.col.max() < self.ncols

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols), dtype=np.float64)
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))
        d[rows, self.col] = self.val
        return d


def from_coo(nrows: int, ncols: int, rows: np.ndarray, cols: np.ndarray,
             vals: np.ndarray | None = None) -> CSR:
    """Sorted CSR from coordinates that are already unique (no duplicate (r, c))."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    if vals is None:
        v = np.ones(len(rows), dtype=np.float64)
    else:
        v = np.asarray(vals, dtype=np.float64)[order]
    counts = np.bincount(rows, minlength=nrows) if nrows > 0 else np.zeros(0, np.int64)
    rp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return CSR(nrows, ncols, rp, cols.astype(np.int32), v)


def with_values(P: CSR, seed: int, lo: float = 0.0, hi: float = 1.0) -> CSR:
    """Copy of pattern P with values iid U[lo, hi) drawn in CSR order."""
    rng = np.random.default_rng(seed)
    v = lo + (hi - lo) * rng.random(P.nnz)
    return CSR(P.nrows, P.ncols, P.row_ptr.copy(), P.col.copy(), v, P.sorted)


def er_poisson(n: int, lam: float, seed: int) -> CSR:
    """BASELINE config 1: n x n, row i has Poisson(lam) nonzeros (clipped to
    [0, n]), columns uniform without replacement, values U[0,1)."""
    rng = np.random.default_rng(seed)
    cnt = np.minimum(rng.poisson(lam, size=n), n).astype(np.int64)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rp[1:])
    col = np.empty(int(rp[-1]), dtype=np.int32)
    for i in range(n):
        c = int(cnt[i])
        if c:
            col[rp[i]:rp[i + 1]] = np.sort(rng.choice(n, size=c, replace=False))
    val = rng.random(int(rp[-1]))
    return CSR(n, n, rp, col, val)


def stencil27(g: int, seed: int, lo: float = 0.5, hi: float = 1.5) -> CSR:
    """BASELINE config 2: 27-point stencil on a g^3 grid, boundary truncated.

    Row id = x + g*(y + g*z); neighbours |dx|,|dy|,|dz| <= 1 inside the grid;
    values iid U[lo, hi) per stored entry in CSR order.
    """
    n = g * g * g
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % g, (idx // g) % g, idx // (g * g)
    rows, cols = [], []
    # enumerate offsets in increasing column order: dz outer, dy, dx inner
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < g) & (y + dy >= 0) & (y + dy < g)
                      & (z + dz >= 0) & (z + dz < g))
                r = idx[ok]
                rows.append(r)
                cols.append(r + dx + g * (dy + g * dz))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    P = from_coo(n, n, rows, cols)
    return with_values(P, seed, lo, hi)


def rmat_edges(scale: int, edge_factor: int, a: float, b: float, c: float,
               seed: int, chunk: int = 1 << 22):
    """Unjittered R-MAT draws: edge_factor * 2^scale draws, each descending
    `scale` levels; quadrant (row bit, col bit) = a:(0,0) b:(0,1) c:(1,0) d:(1,1).
    Returns (rows, cols) int64 arrays with duplicates still present."""
    rng = np.random.default_rng(seed)
    ndraw = edge_factor << scale
    rows = np.zeros(ndraw, dtype=np.int64)
    cols = np.zeros(ndraw, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for s in range(0, ndraw, chunk):
        e = min(ndraw, s + chunk)
        r = np.zeros(e - s, dtype=np.int64)
        q = np.zeros(e - s, dtype=np.int64)
        for lvl in range(scale):
            u = rng.random(e - s)
            rb = u >= ab
            cb = ((u >= a) & (u < ab)) | (u >= abc)
            bit = np.int64(1) << np.int64(scale - 1 - lvl)
            r |= rb.astype(np.int64) * bit
            q |= cb.astype(np.int64) * bit
        rows[s:e] = r
        cols[s:e] = q
    return rows, cols


def _dedup(n: int, rows: np.ndarray, cols: np.ndarray):
    key = np.unique(rows * np.int64(n) + cols)
    return key // n, key % n


def rmat(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19,
         value_seed: int | None = None) -> CSR:
    """BASELINE config 3: R-MAT (G500 seeds by default), duplicates merged, values
    U[0,1) drawn per unique entry in CSR order from `value_seed` (default seed+1)."""
    n = 1 << scale
    r, q = rmat_edges(scale, edge_factor, a, b, c, seed)
    r, q = _dedup(n, r, q)
    P = from_coo(n, n, r, q)
    return with_values(P, seed + 1 if value_seed is None else value_seed)


def symmetrise_pattern(A: CSR, drop_diagonal: bool = False) -> CSR:
    """Pattern of A + A^T with values 1.0 (optionally without self loops)."""
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(A.row_ptr))
    cols = A.col.astype(np.int64)
    rr = np.concatenate([rows, cols])
    cc = np.concatenate([cols, rows])
    if drop_diagonal:
        keep = rr != cc
        rr, cc = rr[keep], cc[keep]
    rr, cc = _dedup(A.nrows, rr, cc)
    return from_coo(A.nrows, A.ncols, rr, cc)


def frontier(n: int, k: int, seed: int) -> CSR:
    """BASELINE config 4's B: n x k, one nonzero (1.0) per column at a uniform row."""
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n, size=k, dtype=np.int64)
    return from_coo(n, k, rows, np.arange(k, dtype=np.int64))


def _tri(A: CSR, lower: bool) -> CSR:
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(A.row_ptr))
    cols = A.col.astype(np.int64)
    keep = cols < rows if lower else cols > rows
    return from_coo(A.nrows, A.ncols, rows[keep], cols[keep], A.val[keep])


def tril_strict(A: CSR) -> CSR:
    return _tri(A, True)


def triu_strict(A: CSR) -> CSR:
    return _tri(A, False)


def identity(n: int) -> CSR:
    return from_coo(n, n, np.arange(n), np.arange(n))


def complete_graph(n: int) -> CSR:
    """K_n adjacency (no self loops), values 1.0."""
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    keep = i != j
    return from_coo(n, n, i[keep], j[keep])


def random_sparse(m: int, n: int, density: float, seed: int, lo=0.0, hi=1.0,
                  empty_rows: float = 0.0) -> CSR:
    """Uniform random pattern (each entry present with prob `density`), values
    U[lo,hi); a fraction `empty_rows` of rows is forced empty."""
    rng = np.random.default_rng(seed)
    if m == 0 or n == 0:
        return CSR(m, n, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    mask = rng.random((m, n)) < density
    if empty_rows > 0:
        mask[rng.random(m) < empty_rows] = False
    r, c = np.nonzero(mask)
    return with_values(from_coo(m, n, r, c), seed + 7919, lo, hi)


def shuffle_within_rows(A: CSR, seed: int) -> CSR:
    """Same matrix, storage order permuted inside every row (reading R11 of
    DESIGN.md for P:378 "column indices ... randomly permuted")."""
    rng = np.random.default_rng(seed)
    key = rng.random(A.nnz)
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(A.row_ptr))
    order = np.lexsort((key, rows))
    return CSR(A.nrows, A.ncols, A.row_ptr.copy(), A.col[order].copy(),
               A.val[order].copy(), sorted=False)


# --------------------------------------------------------------------------
# The five BASELINE.json configurations (seeds fixed here).
# --------------------------------------------------------------------------
WORKLOADS = {
    "c1_er4096": "ER n=4096 Poisson(8) rows, U[0,1); C = A*A sorted",
    "c2_stencil64": "27-point stencil 64^3, U[0.5,1.5); C = A*A",
    "c3_rmat20": "R-MAT s20 ef16 (.57,.19,.19,.05) dedup, U[0,1); C = A*A",
    "c4_tallskinny": "sym R-MAT s20 ef16 pattern x frontier(1024); C = A*B",
    "c5_triangle": "sym R-MAT s20 ef16 no loops; C = L*U, mask by G, count/2",
}


def workload(name: str, scale: int | None = None):
    """Return (A, B, extra) for a named config. `scale` shrinks the R-MAT /
    stencil / ER size for parity tests (same recipe, smaller)."""
    if name == "c1_er4096":
        n = 4096 if scale is None else (1 << scale)
        A = er_poisson(n, 8.0, 1001)
        return A, A, {}
    if name == "c2_stencil64":
        g = 64 if scale is None else scale
        A = stencil27(g, 1002)
        return A, A, {}
    s = 20 if scale is None else scale
    if name == "c3_rmat20":
        A = rmat(s, 16, 1003)
        return A, A, {}
    R = rmat(s, 16, 1003)
    if name == "c4_tallskinny":
        A = symmetrise_pattern(R)
        B = frontier(A.nrows, 1024, 1004)
        return A, B, {}
    if name == "c5_triangle":
        G = symmetrise_pattern(R, drop_diagonal=True)
        return tril_strict(G), triu_strict(G), {"G": G}
    raise KeyError(name)


def crafted_rows(specs, ncols: int, seed: int, shuffle: bool = False):
    """(A, B) whose row i of A*B has exactly flop = specs[i][0] products and
    nnz = specs[i][1] distinct columns (0 <= nnz <= min(flop, ncols); flop > 0
    needs nnz > 0).  Row i of A selects fresh rows of B: q = flop // nnz copies
    of one column set S (|S| = nnz) and one row holding the first flop % nnz
    columns of S.  Used to hit every bin boundary of the GPU path; the values
    are U[0.5, 1.5)."""
    rng = np.random.default_rng(seed)
    a_rows, a_cols, b_rows, b_cols = [], [], [], []
    nb = 0
    for i, (f, n) in enumerate(specs):
        if f == 0:
            continue
        assert 0 < n <= min(f, ncols)
        S = rng.choice(ncols, size=n, replace=False).astype(np.int64)
        q, rem = divmod(f, n)
        lens = [n] * q + ([rem] if rem else [])
        for L in lens:
            a_rows.append(i)
            a_cols.append(nb)
            b_rows.append(np.full(L, nb, np.int64))
            b_cols.append(S[:L])
            nb += 1
    m = len(specs)
    A = from_coo(m, nb, np.array(a_rows, np.int64), np.array(a_cols, np.int64))
    B = from_coo(nb, ncols, np.concatenate(b_rows) if b_rows else np.zeros(0, np.int64),
                 np.concatenate(b_cols) if b_cols else np.zeros(0, np.int64))
    A = with_values(A, seed + 1, 0.5, 1.5)
    B = with_values(B, seed + 2, 0.5, 1.5)
    if shuffle:
        A, B = shuffle_within_rows(A, seed + 3), shuffle_within_rows(B, seed + 4)
    return A, B
